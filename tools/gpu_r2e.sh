cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_bench_configs.py tests/test_measure.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_e.log
timeout 600 python bench.py --config k4 --steps 20 --warmup 3 2>&1 | tail -1
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 2>&1 | tail -1
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
