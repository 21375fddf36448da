mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
PYTHONPATH=. MR_LIB_PATH=variants/prof/libmri_b200.so timeout 300 python scripts/phase_prof.py C4 64 > gpurun_out/phase_c4.log 2>&1; cat gpurun_out/phase_c4.log
PYTHONPATH=. MR_LIB_PATH=variants/prof/libmri_b200.so timeout 300 python scripts/phase_prof.py C5 48 > gpurun_out/phase_c5.log 2>&1; cat gpurun_out/phase_c5.log
