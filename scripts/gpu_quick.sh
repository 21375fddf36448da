# quick check: chemistry parity tests + C4 64^3 bench + phase profile
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "fast_rhs or fixture or full_run or determinism" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q_pytest.log
timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/q_bench.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/q_bench.log').read().strip().split('\n')[-1])
print('C4 64^3 ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), d['time_split_ms'])" || tail -3 gpurun_out/q_bench.log
if [ -f variants/prof/libmri_b200.so ]; then
PYTHONPATH=. MR_LIB_PATH=variants/prof/libmri_b200.so timeout 300 python scripts/phase_prof.py C4 64 2>&1 | tail -8
fi
