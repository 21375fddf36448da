# GPU test pass on one B200: smoke, pytest -m gpu (durations), optional -k filter in $1
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${TAG:-t}
nproc > gpurun_out/host_$TAG.txt; free -g | head -2 >> gpurun_out/host_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 3000 python -m pytest tests -m gpu -q -s --timeout 1500 --durations=25 "${K[@]}" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|error" gpurun_out/pytest_$TAG.log | tail -3
grep -E "max rel err" gpurun_out/pytest_$TAG.log | head -20
