cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/prof gpurun_out/prof_sum
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/prof_sum/r02_launches_c3pre.csv \
  python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --set classification=pre > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/prof_sum/r02_launches_c3pre.csv gpurun_out/prof_sum/r02_launches_c3pre.md > /dev/null
for k in raycast_chain_kernel raycast_chain_coop_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k<" -s 1 -c 1 -o /tmp/prof/pre_$k -f \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --set classification=pre > /dev/null 2>&1; echo "$k rc=$?"
python tools/ncu_summary.py full /tmp/prof/pre_$k.ncu-rep gpurun_out/prof_sum/r02_ncu_c3pre_$k > /dev/null 2>&1
done
