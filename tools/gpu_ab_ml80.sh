# A/B: hand-off threshold 80 samples left (64 for starved frames) vs 64
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do CONFIGS="c3 c2 c1 c4 c3soft" bash tools/variants.sh build_variants/base.so build_variants/ml80.so; done
