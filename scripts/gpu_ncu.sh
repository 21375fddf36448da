# ncu --set full of one chemistry chain launch at C4 physics on 64^3 (arg1 = tag)
mkdir -p gpurun_out
TAG=${1:-chem}
timeout 300 python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-chem_chain} -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
