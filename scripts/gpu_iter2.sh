# parity tests + C4-physics 64^3 timing + one ncu capture of the chemistry kernel
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${1:-it}
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not full_size" -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/b64_$TAG.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b64_$TAG.log').read().strip().split('\n')[-1])
print('ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), d['time_split_ms'])" || tail -5 gpurun_out/b64_$TAG.log
if [ -n "$NCU" ]; then
timeout 300 python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 0 -c 1 -o gpurun_out/prof_$TAG python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
fi
