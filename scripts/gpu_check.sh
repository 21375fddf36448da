mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
python -c "import paper_2211_03293_b200 as P; c=P.Context(0); print('peak fp64 TFLOP/s', c.fp64_peak())" > gpurun_out/peak.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"
tail -3 gpurun_out/*.log
