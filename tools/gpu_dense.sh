# dense-burst A/B: correctness of the unlit paths, then frame rates
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_bench_configs.py -k "stress or c1 or c2" tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -3
bash tools/gpu_ab_variants.sh "c3stress c3 c2" build_variants/burst0.so build_variants/burst8.so build_variants/burst128.so
