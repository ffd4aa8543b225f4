#!/bin/bash
# Round-2 GPU check: full GPU test suite, smoke, headline bench, reference arm.
set -x
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for c in c3 c2 c1 c3soft c3stress c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/bench.jsonl 2>>gpurun_out/bench.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --config c3 --steps 2 --warmup 1 > gpurun_out/bench_ref.jsonl 2>&1; echo "ref rc=$?"
