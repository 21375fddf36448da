# ncu evidence at the benched size (C4 256^3): launch list of a bench run, one
# --set full capture of the first chemistry chain launch and of the first
# stencil launch.  Each ncu command follows a plain run of the same command.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 $CMD > gpurun_out/ncu_plain1.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_256.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
CMD0="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 900 $CMD0 > gpurun_out/ncu_plain0.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 0 -c 1 -o gpurun_out/chem_chain_c4_256 $CMD0 > gpurun_out/ncu_chem.log 2>&1; echo "chem rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:stencil -s 0 -c 1 -o gpurun_out/stencil_c4_256 $CMD0 > gpurun_out/ncu_sten.log 2>&1; echo "stencil rc=$?"
