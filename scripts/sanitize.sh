#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py, one log per tool -> gpurun_out/sanitizer_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
