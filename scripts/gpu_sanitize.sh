# one compute-sanitizer tool over scripts/sanitize_run.py (plain run first)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TOOL=${1:-memcheck}
timeout 600 python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
timeout 3000 compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_run.py > gpurun_out/sanitize_$TOOL.log 2>&1; echo "sanitizer $TOOL rc=$?"
tail -15 gpurun_out/sanitize_$TOOL.log
