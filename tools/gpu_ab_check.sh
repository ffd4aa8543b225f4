# correctness of each library variant (bench-config frames + fuzz), then A/B frame rates
# usage: bash tools/gpu_ab_check.sh "CONFIGS" variant.so ...
cd "$GRAFT_REPO_ROOT"
CF=$1; shift
for l in "" "$@"; do
  echo "== ${l:-base}"; VR_LIB=$l timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
done
bash tools/gpu_ab_variants.sh "$CF" "$@"
