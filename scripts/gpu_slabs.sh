# per-GPU work of the P-GPU slab decomposition on one B200 (bench.py --slab-of P), C4 and C3,
# plus the C4 rank-of-8 slab through the NCCL rank path
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for P in 1 2 4 8; do
  timeout 900 python bench.py --slab-of $P --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/slab_c4_$P.log 2>&1; echo "c4 $P rc=$?"
done
for P in 1 2 4; do
  timeout 900 python bench.py --config C3 --slab-of $P --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/slab_c3_$P.log 2>&1; echo "c3 $P rc=$?"
done
timeout 900 python bench.py --slab-of 8 --nccl-self --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/slab_c4_8_nccl.log 2>&1; echo "c4 8 nccl rc=$?"
