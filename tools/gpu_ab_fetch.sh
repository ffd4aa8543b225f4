# A/B of ray-queue head read variants (build_variants/*.so) + parity of the candidate
VR_LIB=build_variants/v2.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do CONFIGS="c3 c2 c1 c4 c3soft" bash tools/variants.sh build_variants/base.so build_variants/head.so build_variants/v2.so; done
