cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
bash tools/gpu_ab_variants.sh "c3iso c3preint c3pre c3" build_variants/head.so
