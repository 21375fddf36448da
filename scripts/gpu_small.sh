# A/B of library builds on the small configs C1 (32^3) and C2 (64^3)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$L; fi
  for C in C1 C2 C3; do
    timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sm_$C.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/sm_$C.log').read().strip().split('\n')[-1])
print('$L $C ms/step %.3f'%d['ms_per_step'], 'chem frac %.3f'%d['roofline']['frac'], d['time_split_ms'])" || tail -3 gpurun_out/sm_$C.log
  done
done
