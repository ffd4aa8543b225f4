# dram bytes of the ray-cast kernels per library variant (ncu, c3)
for lib in "$@"; do
  VR_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread -k regex:raycast_ -s 6 -c 2 --csv \
    python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(dram|gpu__time|launch)' | awk -F'","' -v l=$lib '{print l, $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200
done
