# long-ray queue threshold (VR_HEAVY_LONG), two passes
for r in 1 2; do KNOB=VR_HEAVY_LONG VALS="256 384 512" CONFIGS="c3 c2 c4 c3soft" bash tools/sweep_knob.sh; done
