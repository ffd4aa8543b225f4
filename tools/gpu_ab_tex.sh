cd "$GRAFT_REPO_ROOT"
VR_LIB=build_variants/tex.so timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py "tests/test_gpu_bench_configs.py::test_c3_stress_window" "tests/test_gpu_bench_configs.py::test_c3_frame" -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for l in "" build_variants/tex.so; do
 for c in c3 c3stress c3soft c2; do
  VR_LIB=$l timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l', d['config']['workload'], round(d['value'],1), round(d['roofline']['kernel_ms'],3))"
 done
done
