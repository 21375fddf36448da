# stencil K2: TMA ring vs cp.async ring (C4 256^3, fast off), then the stencil-touching GPU tests
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "slow_rhs" > gpurun_out/sten_quick.log 2>&1; rc=$?
tail -2 gpurun_out/sten_quick.log
if [ $rc -ne 0 ]; then echo "stencil tests failed, stopping"; exit 1; fi
for L in - variants/notma/libmri_b200.so; do
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$PWD/$L; fi
  echo "lib=$L: $(timeout 600 python scripts/sten_bench.py C4 256 3 2>&1 | tail -1)"
  echo "lib=$L: $(timeout 600 python scripts/sten_bench.py C3 128 3 2>&1 | tail -1)"
done
unset MR_LIB_PATH
TAG=d bash scripts/gpu_tests.sh "slow_rhs or transport or nccl or multidevice or virtual_rank or imex or c3_full"
