cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
VR_LIB=build_variants/sdiv2.so timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -1
bash tools/gpu_ab_variants.sh "c3 c3soft c2 c4 c3iso" build_variants/sdiv2.so
