cd "$GRAFT_REPO_ROOT"
timeout 300 python tools/diag_c2.py 2>&1 | tail -4
timeout 300 python tools/diag_c2.py 512,512,512 1024 soft-tissue blocks 2>&1 | tail -4
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
