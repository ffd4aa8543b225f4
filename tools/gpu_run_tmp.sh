cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/gpu_ab_variants.sh "c3 c3soft c2 c3stress" build_variants/p5.so build_variants/h5.so build_variants/p5h5.so
