# A/B library variants on several configs: bash tools/gpu_ab_variants.sh "c3 c3soft c2" lib1.so lib2.so ...
cd "$GRAFT_REPO_ROOT"
CF=$1; shift
for rep in 1 2; do
for l in "" "$@"; do
 for c in $CF; do
  VR_LIB=$l timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${l:-base}', d['config']['workload'], round(d['value'],1))"
 done
done
done
