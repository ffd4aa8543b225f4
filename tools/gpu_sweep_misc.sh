# runtime knobs around the current defaults, two passes at C3 (+C2/C4 for the hand-off knobs)
for r in 1 2; do
KNOB=VR_HEAVY_LONG VALS="320 384 448" CONFIGS="c3 c4" bash tools/sweep_knob.sh
KNOB=VR_HEAVY_MIN_LEFT VALS="64 80 96" CONFIGS="c3 c2" bash tools/sweep_knob.sh
KNOB=VR_AABB_CTAS VALS="4 8 16" CONFIGS="c3" bash tools/sweep_knob.sh
done
