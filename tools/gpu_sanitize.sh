# compute-sanitizer over tools/sanitize_run.py; logs to gpurun_out/sanitize_*.log
cd /root/repo
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 2400 $CS --tool $tool --print-limit 50 --error-exitcode 99 python tools/sanitize_run.py "$@" \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run: done|Error" gpurun_out/sanitize_$tool.log | head -5
done
