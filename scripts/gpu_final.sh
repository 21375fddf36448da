# Round-end measurements on one B200: the default bench line (C4), the
# reference arm, every other config, the step-size check.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/final_gpu.txt 2>&1
nproc >> gpurun_out/final_gpu.txt; lscpu | grep "Model name" >> gpurun_out/final_gpu.txt; free -g | head -2 >> gpurun_out/final_gpu.txt
timeout 1200 python bench.py > gpurun_out/final_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/final_c4.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_ref.log | cut -c1-300
for C in C1 C2 C3; do
  timeout 900 python bench.py --config $C > gpurun_out/final_$C.log 2>&1; echo "$C rc=$?"; tail -1 gpurun_out/final_$C.log | cut -c1-200
done
timeout 900 python bench.py --config C5 --slab-of 8 > gpurun_out/final_C5.log 2>&1; echo "C5 rc=$?"; tail -1 gpurun_out/final_C5.log | cut -c1-200
timeout 900 python bench.py --slab-of 8 --nccl-self --no-cpu > gpurun_out/final_c4_slab8_nccl.log 2>&1; echo "c4 slab8 nccl rc=$?"
timeout 900 python bench.py --slab-of 8 --no-cpu > gpurun_out/final_c4_slab8.log 2>&1; echo "c4 slab8 rc=$?"
