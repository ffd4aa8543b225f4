# Bounds-checked build over the whole GPU suite, then the release library's frame rates.
# Build first: python paper_2005_01442_b200/_build.py build_variants/bounds.so VR_BOUNDS_CHECK
cd "$GRAFT_REPO_ROOT"
VR_LIB=build_variants/bounds.so timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -2
VR_LIB=build_variants/bounds.so timeout 300 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bounds-checked c3', round(d['value'],1))"
bash tools/gpu_ab_variants.sh "c3 c3soft"
