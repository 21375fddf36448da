# K1 variants: ms/step and state hash (bitwise) at C4 physics 128^3 and C5 64^3
export PYTHONUNBUFFERED=1
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  timeout 300 python scripts/chem_state_hash.py C4 128 2>&1 | tail -1
  timeout 300 python scripts/chem_state_hash.py C5 64 2>&1 | tail -1
done
