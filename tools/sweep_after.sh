# sweep VR_HEAVY_VIS (hand rays over before the queue drains once they composited this many samples)
for c in ${CONFIGS:-c3 c2 c3soft}; do
 for v in ${VALS:-1073741824 32 16 8 4 2}; do
  VR_HEAVY_VIS=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vis=$v', d['config']['workload'], round(d['value'],1), 'fps')"
 done
done
