# bench every BASELINE config on one GPU (C4 is the default bench line)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for C in C1 C2 C3; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --sample-n 16 > gpurun_out/cfg_$C.log 2>&1; echo "$C rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/cfg_$C.log').read().strip().split('\n')[-1])
print('$C', 'ms/step %.3f'%d['ms_per_step'], 'value %.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'chem frac %.3f'%d['roofline']['frac'], 'sten GB/s %.0f'%(d['roofline_stencil']['achieved'] or 0), 'cpu %.3g'%d['cpu_baseline']['value'], d['time_split_ms'], 'launches', d['gpu_launches'])"
done
