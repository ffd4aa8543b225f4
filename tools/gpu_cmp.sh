# [pytest -m gpu with the in-tree library,] then the perf sweep of each variant
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log; }
bash tools/variants.sh build_variants/*.so
