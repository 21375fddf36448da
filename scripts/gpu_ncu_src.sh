# ncu --set full of one C4-physics chemistry chain launch at 64^3 for reaction counts R (args),
# plus the per-CUDA-line source page (stall samples) of each capture
mkdir -p gpurun_out
for R in "$@"; do
  timeout 300 python scripts/chem_time.py C4 64 $R > gpurun_out/plain_r$R.log 2>&1 || { echo "plain R=$R failed"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 3 -c 1 \
     -o gpurun_out/k1_r$R python scripts/chem_time.py C4 64 $R > gpurun_out/ncu_r$R.log 2>&1; echo "ncu R=$R rc=$?"
  ncu -i gpurun_out/k1_r$R.ncu-rep --page source --csv --print-source cuda > gpurun_out/k1_r${R}_src.csv 2>/dev/null
done
