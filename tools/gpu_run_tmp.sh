cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/gpu_ab_variants.sh "c3pre c3preint c3iso" build_variants/cs0.so
