cd "$GRAFT_REPO_ROOT"
VR_LIB=build_variants/simd.so timeout 600 python -m pytest tests/test_measure.py -x -q -m gpu 2>&1 | tail -1
for rep in 1 2; do for l in "" build_variants/simd.so; do
VR_LIB=$l timeout 300 python bench.py --config k4 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${l:-base}', round(r['kernel_ms']*1e3,1), 'count', round(r['count_only']['kernel_ms']*1e3,1), 'balls', round(r['balls_ms']*1e3,1), d['result']['count'], d['result']['S_mm2'])"
done; done
