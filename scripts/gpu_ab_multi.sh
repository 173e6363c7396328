#!/bin/bash
# A/B of env settings: bash scripts/gpu_ab_multi.sh TAG "c3 c2" "K=1,L=2,4" "K=0,L=1,2" ...
# each setting: comma-free groups separated by ';' -> here "A=x;B=y" (use ';' between vars)
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
for rep in $(seq 1 ${REPS:-2}); do for c in $CFGS; do for v in "$@"; do
  name=$(echo "$v" | sed 's/EBIC_//g; s/[;=,]/_/g')
  env $(echo "$v" | tr ';' ' ') timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 5 --no-cpu-baseline > $OUT/ab_${TAG}_${c}_${name}_$rep.json 2>/dev/null
done; done; done
echo done
