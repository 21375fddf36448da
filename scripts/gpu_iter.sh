# quick iteration: GPU parity tests + chemistry layout sweep at C4 physics on 64^3
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not full_size" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for L in ${LAYOUTS:-"16,16,4" "32,8,7" "8,32,2"}; do
  MR_CHEM_BLOCK=$L timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/lay_$L.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lay_$L.log').read().strip().split('\n')[-1])
print('$L', 'ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), d['time_split_ms'])" || tail -5 gpurun_out/lay_$L.log
done
