cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/prof gpurun_out/prof_sum
timeout 600 ncu --set full --clock-control none --import-source on -k regex:raycast_chain -s 1 -c 1 -o /tmp/prof/chain_iso -f \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --set mode=isosurface --set isovalue=600 > /dev/null 2>&1; echo "iso rc=$?"
python tools/ncu_summary.py full /tmp/prof/chain_iso.ncu-rep gpurun_out/prof_sum/r02_ncu_c3iso_raycast_chain_kernel > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:raycast_chain -s 1 -c 1 -o /tmp/prof/chain_pre -f \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --set classification=preintegrated > /dev/null 2>&1; echo "preint rc=$?"
python tools/ncu_summary.py full /tmp/prof/chain_pre.ncu-rep gpurun_out/prof_sum/r02_ncu_c3preint_raycast_chain_kernel > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_sum/r02_launches_c3iso.csv \
  python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --set mode=isosurface --set isovalue=600 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/prof_sum/r02_launches_c3iso.csv gpurun_out/prof_sum/r02_launches_c3iso.md > /dev/null
