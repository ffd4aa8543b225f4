cd "$GRAFT_REPO_ROOT"
bash tools/gpu_ab_variants.sh "c3pre c3preint c3soft c3 c2 c4" build_variants/hv64.so build_variants/hv1073741824.so
