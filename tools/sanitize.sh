#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py: memcheck, racecheck (shared
# memory hazards), synccheck (barrier / warp-sync misuse), initcheck.
# Logs -> gpurun_out/sanitize/<tool>_<case>.log
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in c1 long multi c2; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout ${TMO:-900} $CS --tool $tool $extra --print-limit 50 python tools/sanitize_case.py $case \
        > gpurun_out/sanitize/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize/${tool}_${case}.log | tr '\n' ' ')"
  done
done
