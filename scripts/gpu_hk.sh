# step-size accuracy of every config + K1 A/B (one-cell vs two-cell kernel)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
( python scripts/hcheck.py C1 1 0.5 0.25
  python scripts/hcheck.py C2 1 0.5 0.25
  python scripts/hcheck.py C3 1 0.5 0.25
  python scripts/hcheck.py C4 1 0.5 0.25 0.125
  python scripts/hcheck.py C5 0.5 0.25 0.125 ) > gpurun_out/hcheck.log 2>&1
cat gpurun_out/hcheck.log
for L in - variants/one/libmri_b200.so; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  for n in 128; do
    timeout 600 python bench.py --n $n --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_$n.log 2>&1
    echo "lib=$L n=$n $(tail -1 gpurun_out/ab_$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["time_split_ms"]["chem"]/d["steps"], d["roofline"]["frac"])')"
  done
done
unset MR_LIB_PATH
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c4_chem2.log 2>&1; tail -1 gpurun_out/bench_c4_chem2.log | cut -c1-600
