#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py, one tool per run (run under gpurun).
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t exit $?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case ok' gpurun_out/sanitize_$t.log | tr '\n' ' ')"
done
