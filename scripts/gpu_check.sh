#!/bin/bash
# Round-level GPU call: tests, smoke, bench (+reference arm), 2-rank gloo run of the
# sharded bench path, ncu launch list and one full capture of the hot kernel per config.
# usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu_$TAG.txt 2>&1
nproc >> $OUT/gpu_$TAG.txt; lscpu | grep "Model name" >> $OUT/gpu_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu -rs > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
for sh in replica rows pop; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
      bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --shard $sh > $OUT/bench_gloo2_${sh}_$TAG.json 2> $OUT/bench_gloo2_${sh}_$TAG.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --shard rows --exchange nccl > $OUT/bench_gloo2_rows_allreduce_$TAG.json 2> $OUT/bench_gloo2_rows_allreduce_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.log 2>&1
for c in c3 c2 c4 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab_|table_count" -s 5 -c 1 \
      -o $OUT/prof_${c}_$TAG -f python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_${c}_$TAG.log 2>&1
done
for c in c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
done
# the slab kernel (no index) on c3 for comparison, and its ncu capture
timeout 600 python bench.py --config c3 --path plane --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_plane_$TAG.json 2> $OUT/bench_c3_plane_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab_" -s 5 -c 1 \
    -o $OUT/prof_c3_plane_$TAG -f python bench.py --config c3 --path plane --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_c3_plane_$TAG.log 2>&1
# index build kernel
timeout 900 ncu --set full --clock-control none -k regex:"build_pair_table" -c 1 \
    -o $OUT/prof_c3_build_$TAG -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python scripts/run_e2e.py > $OUT/run_e2e_$TAG.txt 2>&1

# keep gpurun_out under the 64 MiB merge cap: raw-page CSVs of every capture,
# the .ncu-rep files only for the C3 kernels
for f in $OUT/prof_*_$TAG.ncu-rep; do
  [ -f "$f" ] || continue
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>/dev/null
  case "$f" in
    *prof_c3_$TAG.ncu-rep|*prof_c3_plane_$TAG.ncu-rep) ;;
    *) rm -f "$f" ;;
  esac
done
du -sh $OUT
# memory / race checking of every kernel family, and the ingest benchmark
bash scripts/gpu_sanitize.sh $TAG
timeout 900 python scripts/ingest_bench.py > $OUT/ingest_$TAG.txt 2>&1
echo done
