#!/bin/bash
# compute-sanitizer over scripts/sanitize_drive.py (run on the GPU box via gpurun);
# one log per tool under gpurun_out/, a summary line per tool on stdout.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1200 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 python scripts/sanitize_drive.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
