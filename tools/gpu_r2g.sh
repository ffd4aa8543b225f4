cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_measure.py tests/test_gpu_bench_configs.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 600 python bench.py --config k4 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('k4', round(r['kernel_ms'],4), 'ms', round(r['frac'],3), 'balls', round(r['balls_ms'],4), r['count_only'], d['result'])"
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value'],1), round(d['ms_per_step'],2), d['samples_taken'])"
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value'],1))"
