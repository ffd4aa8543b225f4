# ncu --set full of the per-frame visibility kernels (AABB fit, setup) at C3
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_c3.log 2>&1 || { echo "plain run failed"; exit 1; }
for k in aabb_kernel vis_setup_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -f -o gpurun_out/prof_setup_$k $CMD > gpurun_out/ncu_setup_$k.log 2>&1; echo $k=$?
done
