# A/B of library builds on C4 physics 64^3 (and C5 slab 16 planes of 384^2 if C5=1)
# usage: bash scripts/gpu_ablibs.sh lib1.so lib2.so ...   ("-" = in-tree build)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "fast_rhs or fixture or full_run or determinism" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab_pytest.log
i=0
for L in "$@"; do
  i=$((i+1))
  if [ "$L" = "-" ]; then unset MR_LIB_PATH; else export MR_LIB_PATH=$L; fi
  timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_$i.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().split('\n')[-1])
print('$L', 'C4 64^3 ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" || tail -3 gpurun_out/ab_$i.log
  if [ -n "$C5" ]; then
  timeout 300 python bench.py --config C5 --n 192 --slab-of 12 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab5_$i.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab5_$i.log').read().strip().split('\n')[-1])
print('$L', 'C5 16x192^2 ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" || tail -3 gpurun_out/ab5_$i.log
  fi
done
unset MR_LIB_PATH
if [ -f variants/prof/libmri_b200.so ]; then
PYTHONPATH=. MR_LIB_PATH=variants/prof/libmri_b200.so timeout 300 python scripts/phase_prof.py C4 64 2>&1 | tail -8
fi
