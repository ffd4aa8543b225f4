# sweep an env knob: KNOB=VR_HEAVY_MIN_LEFT VALS="32 64 128" CONFIGS="c3 c2" bash tools/sweep_knob.sh
for c in ${CONFIGS:-c3 c2 c3soft}; do
 for v in $VALS; do
  env $KNOB=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KNOB=$v', d['config']['workload'], round(d['value'],1), 'fps')"
 done
done
