mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$L; fi
  echo "== $L"
  timeout 300 python scripts/sten_bench.py C4 256 2 2>&1 | tail -1
  timeout 300 python scripts/sten_bench.py C3 128 3 2>&1 | tail -1
  timeout 300 python scripts/sten_bench.py C2 64 3 2>&1 | tail -1
done
