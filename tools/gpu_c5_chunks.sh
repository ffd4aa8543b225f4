cd "$GRAFT_REPO_ROOT"
for l in build_variants/c1.so build_variants/nd4.so build_variants/nd16.so build_variants/nd64.so build_variants/d4.so ""; do
VR_LIB=$l timeout 300 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $l', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"
done
