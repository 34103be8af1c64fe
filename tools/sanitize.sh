#!/bin/bash
# compute-sanitizer over every sweep kernel variant at small shapes.
# Run on a GPU box:  bash tools/sanitize.sh  -> gpurun_out/sanitize/<tool>.log
O=gpurun_out/sanitize
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = initcheck ] && extra=""
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
done
