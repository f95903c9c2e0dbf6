#!/bin/bash
# compute-sanitizer over scripts/sanitize_drive.py: memcheck, racecheck, synccheck, initcheck.
# Logs under gpurun_out/$TAG; one line per tool with its error summary.
TAG=${1:-san}
mkdir -p gpurun_out/$TAG
for tool in memcheck racecheck synccheck initcheck; do
  for part in eval ga brute; do
    extra=""; [ $tool = synccheck ] && extra="--num-cuda-barriers 16384"
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 20 python scripts/sanitize_drive.py $part > gpurun_out/$TAG/${tool}_$part.txt 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|driver done' gpurun_out/$TAG/${tool}_$part.txt | tr '\n' ' ')"
  done
done
