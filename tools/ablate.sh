run() { timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['desc'][-60:], round(d['value'],1), 'fps', round(d['roofline']['kernel_ms'],3), 'ms', d['interpolated_samples'], d['march_iterations'])"; }
run --config c3
run --config c3 --set lighting=false
run --config c3 --set interpolation=trilinear
run --config c3 --set early_termination_alpha=1.0
run --config c3 --set use_blocks=false
