# compare library variants: bash tools/variants.sh build_variants/*.so  (CONFIGS="c3 c2" to narrow)
for lib in "$@"; do
  for c in ${CONFIGS:-c3 c3soft c2 c3stress}; do
    VR_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms', 'interp', d.get('interpolated_samples'), 'iters', d.get('march_iterations'))" || echo "$lib $c failed"
  done
done
