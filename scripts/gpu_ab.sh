#!/bin/bash
# A/B of an env knob on the same box: bash scripts/gpu_ab.sh TAG VAR "v1 v2" "configs"
TAG=$1; VAR=$2; VALS=$3; CFGS=${4:-"c3 c4"}
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do for c in $CFGS; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ab_${TAG}_${c}_${VAR}${v}_$rep.json 2>/dev/null
done; done; done
echo done
