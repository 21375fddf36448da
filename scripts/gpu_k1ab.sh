# K1 library-variant A/B on C4 physics at 128^3 (ms per step, failure-tolerant timer)
export PYTHONUNBUFFERED=1
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  timeout 300 python scripts/chem_time.py C4 128 2>&1 | tail -1
done
