# ncu --set full of one kernel (regex $K, default raycast_heavy) for each library variant, config $C (default c3)
K=${K:-raycast_heavy}; C=${C:-c3}
for lib in "$@"; do
  n=$(basename $lib .so)
  VR_LIB=$lib timeout 600 ncu --set full --import-source on -k regex:$K -s 3 -c 1 -f -o gpurun_out/var_${n}_$C \
    python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}.log 2>&1; echo $n=$?
done
