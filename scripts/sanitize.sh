#!/bin/bash
# compute-sanitizer over every entry point (scripts/sanitize.py); one log per tool.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY\|Error\|Hazard' gpurun_out/sanitize_$tool.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
