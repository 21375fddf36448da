# A/B timing of env settings on C4 physics at 64^3: each arg = "NAME=VAL" or "-"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
i=0
for E in "$@"; do
  i=$((i+1))
  if [ "$E" = "-" ]; then EV=""; else EV="$E"; fi
  env $EV timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_$i.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().split('\n')[-1])
print('$E', 'ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" || tail -3 gpurun_out/ab_$i.log
done
