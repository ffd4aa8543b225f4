cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/prof gpurun_out/prof_sum
for k in threshold_kernel inside_bits_kernel straddle_scan_kernel cell_area_kernel ball_surface_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o /tmp/prof/k4_$k -f \
    python bench.py --config k4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "$k rc=$?"
  python tools/ncu_summary.py full /tmp/prof/k4_$k.ncu-rep gpurun_out/prof_sum/r02_ncu_k4_$k > /dev/null 2>&1
  ncu -i /tmp/prof/k4_$k.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for name in ['gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__thread_inst_executed_per_inst_executed.ratio']:
    if name in h: print('$k', name, v[h.index(name)], rows[1][h.index(name)])
"
done
