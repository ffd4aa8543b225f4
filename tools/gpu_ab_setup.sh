timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
CONFIGS="c3 c2 c1 c4" bash tools/variants.sh build_variants/head.so build_variants/setup1.so build_variants/head.so build_variants/setup1.so
