#!/bin/bash
# compute-sanitizer passes over a small GPU workload per kernel family.  usage: tools/gpu_sanitize.sh tag
OUT=gpurun_out/$1; mkdir -p $OUT
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 99 $EXTRA \
    python tools/sanitize_workload.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/$tool.log >> $OUT/summary.txt
done
cat $OUT/summary.txt
