#!/bin/bash
# compute-sanitizer over the small all-kernel workload (tools/sanitize.py)
set -u
OUT=gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok" $OUT/sanitize_$tool.log | tail -3
done
