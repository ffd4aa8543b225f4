timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for r in 1 2; do bash tools/gpu_knob.sh VR_NO_PDL "c3 c2 c1 c4"; done
for v in 0 1; do VR_NO_PDL=$v timeout 300 python bench.py --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_PDL=$v e2e', d['value'], d['e2e']['value'])"; done
