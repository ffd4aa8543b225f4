cd "$GRAFT_REPO_ROOT"
bash tools/gpu_ab_variants.sh "c3 c3soft c2" build_variants/hs0.so build_variants/hs1.so
