for m in 0 64 128 192 256 384 512; do
  for c in c3 c3soft c2; do
    VR_HEAVY_MIN_LEFT=$m timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('min_left=$m', d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms')"
  done
done
