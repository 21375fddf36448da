mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "slow_rhs or virtual or full_run or transport" > gpurun_out/pytest_sten.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sten.log
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_sten.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_sten.log').read().strip().split('\n')[-1])
print('ms/step %.1f'%d['ms_per_step'], 'stencil', d['roofline_stencil'], d['time_split_ms'])"
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:stencil -s 0 -c 1 -o gpurun_out/prof_sten25 python bench.py --n 128 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_sten25.log 2>&1; echo "ncu rc=$?"
fi
