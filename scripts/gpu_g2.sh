# two-group chemistry kernel: GPU tests, then A/B against the single-group build
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g2_pytest.log
bash scripts/gpu_ab.sh "C4 128" - variants/g1/libmri_b200.so
bash scripts/gpu_ab.sh "C5 128" - variants/g1/libmri_b200.so
