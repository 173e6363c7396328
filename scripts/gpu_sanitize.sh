#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r1}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > $OUT/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool exit $?" >> $OUT/sanitize_${tool}_$TAG.log
done
echo done
