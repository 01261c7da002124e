#!/bin/bash
# compute-sanitizer over every kernel family (run under gpurun):
#   bash tools/sanitize.sh TAG   -> gpurun_out/sanitizer_TAG.txt
TAG=${1:-r02}
OUT=gpurun_out/sanitizer_$TAG.txt
: > $OUT
python tools/sanitize_cases.py >> $OUT 2>&1; echo "plain rc=$?" >> $OUT
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool ===" >> $OUT
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --target-processes all \
      python tools/sanitize_cases.py >> $OUT 2>&1
  echo "$tool rc=$?" >> $OUT
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=" $OUT | tail -2
done
