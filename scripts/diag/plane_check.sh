# slab (plane path) kernel check: parity of every pair layout, C3 plane bench, shared-memory wavefronts
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pair_layout or plane or zero_copy" > gpurun_out/plane_tests_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/plane_tests_$TAG.log
for i in 1 2; do
  timeout 300 python bench.py --config c3 --path plane --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/plane_bench_${TAG}_$i.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread \
  --clock-control none -k regex:"slab_pair" -s 3 -c 1 --csv python bench.py --config c3 --path plane --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plane_ncu_$TAG.csv 2>/dev/null
