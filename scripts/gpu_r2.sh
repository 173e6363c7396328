#!/bin/bash
# Round-2 GPU call: tests, smoke, default bench, reference arm, c2/c4/c5 lines,
# sweep, launch list and one full ncu capture of the count kernel.
# usage (repo root, on the GPU box): bash scripts/gpu_r2.sh [tag] [skip_tests]
set -u
TAG=${1:-r2}
SKIP_TESTS=${2:-0}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu_$TAG.txt 2>&1
nproc >> $OUT/gpu_$TAG.txt
if [ "$SKIP_TESTS" = "0" ]; then
  timeout 1800 python -m pytest tests -q -m gpu -rs > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
for c in c2 c4 c5 spec; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
done
timeout 600 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench_c3_200_$TAG.json 2> $OUT/bench_c3_200_$TAG.err
timeout 600 python bench.py --config c3 --path plane --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_plane_$TAG.json 2> $OUT/bench_c3_plane_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"table_count|lazy" -s 5 -c 1 \
    -o $OUT/prof_c3_$TAG -f python bench.py --config c3 --steps 2 --warmup 5 --no-cpu-baseline > $OUT/ncu_full_c3_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"table_count_warp_multi" -s 12 -c 1 \
    -o $OUT/prof_c4_$TAG -f python bench.py --config c4 --steps 2 --warmup 5 --no-cpu-baseline > $OUT/ncu_full_c4_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"build_pair_table" -c 1 \
    -o $OUT/prof_c3_build_$TAG -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"table_count_group" -s 3 -c 1 \
    -o $OUT/prof_sweep1k_$TAG -f python bench.py --sweep --sweep-r 1000 --sweep-l 5 --no-cpu-baseline > /dev/null 2>&1
for f in $OUT/prof_*_$TAG.ncu-rep; do
  [ -f "$f" ] || continue
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>/dev/null
  case "$f" in *prof_c3_$TAG.ncu-rep) ;; *) rm -f "$f" ;; esac
done
timeout 1200 python bench.py --sweep --no-cpu-baseline > $OUT/sweep_$TAG.jsonl 2> $OUT/sweep_$TAG.err
du -sh $OUT
echo done
