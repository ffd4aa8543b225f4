# A/B: hand-off of freshly started rays once the ray queue has drained (build_variants/*.so)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do CONFIGS="c3 c2 c1 c4 c3soft c3stress" bash tools/variants.sh build_variants/base.so build_variants/p3.so; done
