#!/bin/bash
# Round-2 profiles: launch lists and ncu --set full captures, summarised on the
# box (the reports themselves are too large to bring back): gpurun_out/prof_sum.
# Usage: bash tools/gpu_prof_r2.sh [TAG] [CONFIGS...]   (default: k4 c3 c3soft c3stress)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r02}; shift
CFGS=${@:-k4 c3 c3soft c3stress}
mkdir -p /tmp/prof gpurun_out/prof_sum
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in $CFGS; do
  extra="--no-e2e"; [ "$c" = k4 ] && extra=""
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file /tmp/prof/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline $extra > /dev/null 2>&1; echo "$c launches rc=$?"
  python tools/ncu_summary.py launches /tmp/prof/launches_$c.csv gpurun_out/prof_sum/${TAG}_launches_$c.md > /dev/null
  cp /tmp/prof/launches_$c.csv gpurun_out/prof_sum/${TAG}_launches_$c.csv
  if [ "$c" = k4 ]; then ks="inside_bits_kernel surface_kernel ball_surface_kernel threshold_kernel"; else ks="raycast_post_kernel raycast_heavy_kernel"; fi
  for k in $ks; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/prof/${c}_$k -f \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline $extra > /dev/null 2>&1; echo "$c $k rc=$?"
    python tools/ncu_summary.py full /tmp/prof/${c}_$k.ncu-rep gpurun_out/prof_sum/${TAG}_ncu_${c}_$k > /dev/null 2>&1
  done
done
ls gpurun_out/prof_sum
