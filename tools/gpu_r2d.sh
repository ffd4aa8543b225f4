cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu4.log
for c in c3 c3soft c2; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms')"; done
