# pipelined host upload: host-buffer parity tests, then the C4 bench line (e2e)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "host_buffer" > gpurun_out/e2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/e2e_pytest.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/e2e_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/e2e_bench.log').read().strip().splitlines()[-1])
print('value %.4g ms/step %.1f e2e %.4g e2e ms/step %.1f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step']))"
