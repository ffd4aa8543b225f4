# Round-end capture: tests, smoke, bench lines for every config + the reference arm,
# launch list and ncu --set full of the ray-cast kernels and the AABB fit at C3.
set -o pipefail
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
: > gpurun_out/final.jsonl
timeout 600 python bench.py 2>gpurun_out/final_err.log | tail -1 >> gpurun_out/final.jsonl; echo c3=$?
for c in c1 c2 c3soft c3stress c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 2>>gpurun_out/final_err.log | tail -1 >> gpurun_out/final.jsonl; echo $c=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>>gpurun_out/final_err.log | tail -1 >> gpurun_out/final.jsonl; echo ref=$?
bash tools/gpu_profile.sh c3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aabb_kernel -s 3 -c 1 -f \
  -o gpurun_out/prof_c3_aabb_kernel python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c3_aabb.log 2>&1; echo aabb=$?
