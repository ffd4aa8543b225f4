cd "$GRAFT_REPO_ROOT"
for l in build_variants/k4_lb4.so build_variants/k4_lb1.so; do
VR_LIB=$l timeout 600 python bench.py --config k4 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', round(r['kernel_ms'],4), 'ms', round(r['frac'],3), 'balls', round(r['balls_ms'],4), d['result'])"
done
VR_LIB=build_variants/k4_lb4.so timeout 1200 python -m pytest tests/test_measure.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
VR_LIB=build_variants/k4_lb4.so timeout 900 python bench.py --config c5 --steps 3 --warmup 2 2>&1 | tail -1
