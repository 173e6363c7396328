#!/bin/bash
# Fast iteration call: GPU tests, c3 bench, c3 ncu capture of the hot kernel.
set -u
TAG=${1:-it}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
for c in c3 c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab_" -s 5 -c 1 \
    -o $OUT/prof_c3_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo done
timeout 300 python scripts/e2e_probe.py > $OUT/e2e_probe_$TAG.log 2>&1
