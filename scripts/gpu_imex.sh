mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_imex.py -q -x --timeout 600 > gpurun_out/pytest_imex.log 2>&1; echo "imex rc=$?"; tail -15 gpurun_out/pytest_imex.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "not full_size and not imex" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
