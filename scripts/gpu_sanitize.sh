#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_cases.py):
# memcheck, racecheck (shared memory), synccheck (barriers), initcheck.
# One log per tool under gpurun_out/; the ERROR SUMMARY lines go to
# gpurun_out/sanitize_summary.txt.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  T0=$(date +%s)
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python scripts/sanitize_cases.py ${PFE_SAN_CASES:-} > gpurun_out/sanitize_$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc wall=$(( $(date +%s) - T0 ))s: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
