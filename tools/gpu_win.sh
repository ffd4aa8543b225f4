timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c3 c2 c3soft c1; do
 for nw in 0 1; do
  VR_NO_WINDOW=$nw timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nowin=$nw', d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms', 'interp', d.get('interpolated_samples'), 'taken', d['samples_taken'])"
 done
done
