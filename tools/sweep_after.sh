for h in 1073741824 512 256 128 64 32; do
  for c in c3 c3soft c2 c3stress; do
    VR_HEAVY_AFTER=$h timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('after=$h', d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms')"
  done
done
