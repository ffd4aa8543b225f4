# A/B: hand-off threshold 128 samples left (64 when the frame is starved) vs the previous commit
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do CONFIGS="c3 c2 c1 c4 c3soft c3stress" bash tools/variants.sh build_variants/base.so build_variants/p5.so; done
VR_HEAVY_MIN_LEFT=192 CONFIGS="c3 c2 c4" bash tools/variants.sh build_variants/p5.so
