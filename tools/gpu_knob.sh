# A/B of an env knob: bash tools/gpu_knob.sh KNOB "c3 c2 ..."
K=$1; CS=${2:-c3 c2 c3soft c1}
for c in $CS; do
 for v in 0 1; do
  env $K=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$K=$v', d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms', 'interp', d.get('interpolated_samples'), 'iters', d.get('march_iterations'))"
 done
done
