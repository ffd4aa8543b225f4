# scratch A/B driver used during tuning: edit the config list and variant libraries, then
#   gpurun -- 'bash tools/gpu_run_tmp.sh'
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
bash tools/gpu_ab_variants.sh "c3 c3soft c2 c4" "$@"
