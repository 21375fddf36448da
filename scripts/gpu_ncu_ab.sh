# ncu --set full of the first chemistry chain launch, C4 physics at 64^3, for
# the current library and an A/B variant library (MR_LIB_PATH)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CMD="python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e"
for L in "${@:-variants/one/libmri_b200.so}" -; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; TAG=cur; else export MR_LIB_PATH=$PWD/$L; TAG=$(basename $(dirname $L)); fi
  timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:chem -s 0 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
done
