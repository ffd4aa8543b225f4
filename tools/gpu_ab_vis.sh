# A/B: visibility bits alongside the setup CTA (build_variants/base.so = previous commit)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
VR_NO_PDL=1 timeout 600 python -m pytest tests -m gpu -x -q -k "visib or block or golden" 2>&1 | tail -1
for r in 1 2; do CONFIGS="c3 c2 c4" bash tools/variants.sh build_variants/base.so build_variants/p4.so; done
