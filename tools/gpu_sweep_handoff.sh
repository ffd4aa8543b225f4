# hand-off knobs after the first-trip rule (runtime env knobs, no rebuild)
KNOB=VR_HEAVY_MIN_LEFT VALS="48 64 96 128" CONFIGS="c3 c2 c1 c3soft" bash tools/sweep_knob.sh
KNOB=VR_HEAVY_LONG VALS="128 256 384" CONFIGS="c3 c2" bash tools/sweep_knob.sh
KNOB=VR_HEAVY_VIS_ALPHA VALS="0.3 0.5 0.7" CONFIGS="c3 c3soft" bash tools/sweep_knob.sh
KNOB=VR_HEAVY_VIS VALS="2 4 8" CONFIGS="c3 c3soft" bash tools/sweep_knob.sh
