#!/bin/bash
# A/B of the packed-pair layouts (EBIC_PAIR_LAYOUT="P,SUB") per config, 2 reps.
TAG=${1:-lay}; CFGS=${2:-"c3 c2 c4 c5"}; LAYS=${3:-"2,4 1,2 2,2 1,1 2,1 1,4"}
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do for c in $CFGS; do for v in $LAYS; do
  EBIC_PAIR_LAYOUT=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ab_${TAG}_${c}_${v/,/_}_$rep.json 2>/dev/null
done; done; done
echo done
