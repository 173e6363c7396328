mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pdl_tests.log 2>&1; echo "exit $?" >> gpurun_out/pdl_tests.log
for p in 1 0 1 0; do
  EBIC_PDL=$p timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null > /tmp/b.json
  python -c "import json; d=json.loads(open('/tmp/b.json').readline()); print('pdl', $p, d['value'], d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/pdl_c4.log
done
