mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -k "reductions or fast_rhs" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
for L in "32,2" "16,4" "16,2"; do
  MR_CHEM_LAYOUT=$L timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c4n64_$L.log 2>&1; echo "layout $L rc=$?"
done
timeout 300 python bench.py --n 64 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4n64.csv python bench.py --n 64 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/prof_chain_c4n64 python bench.py --n 64 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 1 -c 1 -o gpurun_out/prof_stencil_c4n64 python bench.py --n 64 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo "ncu3 rc=$?"
