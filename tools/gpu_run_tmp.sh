cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_measure.py -x -q -m gpu 2>&1 | tail -1
VR_LIB=build_variants/k4u8.so timeout 600 python -m pytest tests/test_measure.py -x -q -m gpu 2>&1 | tail -1
for rep in 1 2; do for l in "" build_variants/k4u8.so build_variants/k4u2.so; do
VR_LIB=$l timeout 300 python bench.py --config k4 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${l:-base}', round(r['kernel_ms']*1e3,1), round(r['frac'],3), 'count', round(r['count_only']['kernel_ms']*1e3,1), round(r['count_only']['frac'],3), 'balls', round(r['balls_ms']*1e3,1))"
done; done
