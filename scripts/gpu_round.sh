# Milestone run on one B200: GPU tests, smoke, default bench (C4), reference
# arm, ncu launch list + one full capture of the chemistry kernel.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep "Model name" >> gpurun_out/gpu_$TAG.txt; free -g | head -2 >> gpurun_out/gpu_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
if [ -z "$NONCU" ]; then
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain64_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 0 -c 1 -o gpurun_out/prof_chem_$TAG python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_chem_$TAG.log 2>&1; echo "ncu chem rc=$?"
ncu --set full --clock-control none --import-source on -k regex:stencil -s 0 -c 1 -o gpurun_out/prof_sten_$TAG python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_sten_$TAG.log 2>&1; echo "ncu stencil rc=$?"
fi
