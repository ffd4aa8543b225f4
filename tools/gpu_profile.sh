# Launch list + ncu --set full of both ray-cast kernels for one config (default c3).
# Each ncu pass runs only after the same command exited 0 without ncu.
C=${1:-c3}
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$C.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$C.log; exit 1; }
tail -1 gpurun_out/plain_$C.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$C.csv $CMD > gpurun_out/ncu_launch_$C.log 2>&1; echo launches=$?
for k in raycast_post_kernel raycast_heavy_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -f -o gpurun_out/prof_${C}_$k $CMD > gpurun_out/ncu_full_${C}_$k.log 2>&1; echo $k=$?
done
