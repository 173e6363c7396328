#!/bin/bash
TAG=${1:-x}; OUT=gpurun_out; mkdir -p $OUT
for c in ${2:-c3 c2 c5}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${c}_$TAG.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
echo done
