# A/B of library variants (MR_LIB_PATH) on one workload: ms per step and the
# chemistry share.  Usage: bash scripts/gpu_ab.sh "C4 128" lib1 lib2 ... ("-" = in-tree)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
read CFG N <<< "$1"; shift
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  timeout 600 python bench.py --config $CFG --n $N --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab.log 2>&1
  echo "$CFG n=$N lib=$L: $(tail -1 gpurun_out/ab.log | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print("ms/step %.1f chem ms/step %.1f frac %.3f" % (d["ms_per_step"], d["time_split_ms"]["chem"]/d["steps"], d["roofline"]["frac"]))
except Exception as e: print("FAILED", e)')"
done
