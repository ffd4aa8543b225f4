cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/prof gpurun_out/prof_sum
for l in default tex; do
  lib=""; [ $l = tex ] && lib=build_variants/tex.so
  VR_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:raycast_post_kernel -s 3 -c 1 -o /tmp/prof/ab_$l -f \
     python bench.py --config c3stress --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$l rc=$?"
  python tools/ncu_summary.py full /tmp/prof/ab_$l.ncu-rep gpurun_out/prof_sum/r02_ab_sampler_${l}_c3stress > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:raycast_kernel -s 1 -c 1 -o /tmp/prof/iso -f \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --set mode=isosurface --set isovalue=600 > /dev/null 2>&1; echo "iso rc=$?"
python tools/ncu_summary.py full /tmp/prof/iso.ncu-rep gpurun_out/prof_sum/r02_ncu_c3iso_raycast_kernel > /dev/null 2>&1
ls gpurun_out/prof_sum | grep -E "ab_|iso"
