# bench contract checks on one GPU: default line, reference arm, 2-rank gloo path, c5, c4
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo default=$?; tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo > gpurun_out/bench_gloo2.log 2>&1; echo gloo2=$?; grep metric gpurun_out/bench_gloo2.log | cut -c1-300
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?; tail -1 gpurun_out/bench_c5.log | cut -c1-300
timeout 600 python bench.py --config c4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -1 gpurun_out/bench_c4.log | cut -c1-300
