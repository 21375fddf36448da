# e2e of library variants (pipelined host step chunk counts) on the C4 bench line
export PYTHONUNBUFFERED=1
for L in "$@"; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/e2e_ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_ab.log').read().strip().splitlines()[-1])
print('$L', 'value %.4g ms/step %.1f e2e %.4g e2e ms/step %.1f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step']))" || tail -3 gpurun_out/e2e_ab.log
done
