# bench every BASELINE config on one GPU (C4 is the default bench line; C5 = one
# rank's slab of the 8-GPU run)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for C in C1 C2 C3; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --sample-n 16 > gpurun_out/cfg_$C.log 2>&1; echo "$C rc=$?"
done
timeout 900 python bench.py --config C5 --slab-of 8 --steps 2 --warmup 1 --e2e-steps 1 --sample-n 16 > gpurun_out/cfg_C5.log 2>&1; echo "C5 rc=$?"
for C in C1 C2 C3 C5; do
  python -c "
import json; d=json.loads(open('gpurun_out/cfg_$C.log').read().strip().split('\n')[-1])
print('$C', 'ms/step %.3f'%d['ms_per_step'], 'value %.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'chem frac %.3f'%d['roofline']['frac'], 'sten frac %.3f'%(d['roofline_stencil']['frac'] or 0), 'cpu %.3g'%d['cpu_baseline']['value'], 'launches', d['gpu_launches'])"
done
