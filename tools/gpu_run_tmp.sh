cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/gpu_ab_variants.sh "c3 c3soft c2 c4 c1" build_variants/cg0.so
