# layout sweep of the chemistry kernel on C4 physics at 64^3 (env MR_CHEM_BLOCK)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not full_size" -x > gpurun_out/pytest_lay.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_lay.log
for L in ${LAYOUTS:-"16,4" "8,7"}; do
  MR_CHEM_BLOCK=$L timeout 300 python bench.py --n 64 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/lay_$L.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lay_$L.log').read().strip().split('\n')[-1])
print('$L', 'ms/step %.2f'%d['ms_per_step'], 'chem TF %.2f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), d['time_split_ms'])" || tail -5 gpurun_out/lay_$L.log
done
if [ -n "$NCU" ]; then
MR_CHEM_BLOCK=$NCU timeout 300 python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain_lay.log 2>&1 && \
MR_CHEM_BLOCK=$NCU ncu --set full --clock-control none --import-source on -k regex:chem_chain -s 0 -c 1 -o gpurun_out/prof_lay python bench.py --n 64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_lay.log 2>&1; echo "ncu rc=$?"
fi
