# warp-specialised chemistry kernel: quick parity, then A/B of serial-warp counts vs the single-group build
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_baseline_sizes.py -x -q --timeout 600 -k "c4_c5_physics" > gpurun_out/ws_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ws_pytest.log
for L in variants/g1 variants/ws1 variants/ws2 variants/ws4; do
  MR_LIB_PATH=$PWD/$L/libmri_b200.so python scripts/chem_time.py C4 128
done
