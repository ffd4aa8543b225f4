# everything the driver runs at round end, plus the other arms/configs
set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu-baseline 2>&1 | grep '^{' | cut -c1-300
for c in c4 c5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200; done
