# Round-2 final measurements on one B200: bench lines (C4 default + reference
# arm + the other configs + C4 slab-of-8 plain / NCCL path), then the ncu
# launch list and --set full captures of K1 and K2 at 256^3.  Each ncu command
# follows a plain run of the same command.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/final_gpu.txt 2>&1
nproc >> gpurun_out/final_gpu.txt; lscpu | grep "Model name" >> gpurun_out/final_gpu.txt; free -g | head -2 >> gpurun_out/final_gpu.txt
timeout 1200 python bench.py > gpurun_out/final_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"
for C in C1 C2 C3; do
  timeout 900 python bench.py --config $C > gpurun_out/final_$C.log 2>&1; echo "$C rc=$?"
done
timeout 900 python bench.py --config C5 --slab-of 8 > gpurun_out/final_C5.log 2>&1; echo "C5 rc=$?"
timeout 900 python bench.py --slab-of 8 --nccl-self --no-cpu > gpurun_out/final_c4_slab8_nccl.log 2>&1; echo "c4 slab8 nccl rc=$?"
timeout 900 python bench.py --slab-of 8 --no-cpu > gpurun_out/final_c4_slab8.log 2>&1; echo "c4 slab8 rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 $CMD > gpurun_out/ncu_plain1.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_256.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
CMD0="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 900 $CMD0 > gpurun_out/ncu_plain0.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 0 -c 1 -o gpurun_out/chem_chain_c4_256 $CMD0 > gpurun_out/ncu_chem.log 2>&1; echo "chem rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:stencil -s 0 -c 1 -o gpurun_out/stencil_c4_256 $CMD0 > gpurun_out/ncu_sten.log 2>&1; echo "stencil rc=$?"
