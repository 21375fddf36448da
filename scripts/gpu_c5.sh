mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 900 python bench.py --config C5 --slab-of 8 --steps 2 --warmup 1 --e2e-steps 1 --sample-n 16 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"; tail -2 gpurun_out/bench_c5.log | cut -c1-3000
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-600
