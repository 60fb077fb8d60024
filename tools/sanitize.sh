# compute-sanitizer over tools/sanitize_cases.py (run under gpurun, one GPU); logs in gpurun_out/
mkdir -p gpurun_out/sanitize
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize/$tool.log
done
