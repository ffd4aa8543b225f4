# full GPU suite, then ncu --set full of the named kernels of one config (summarised on the box)
# usage: bash tools/gpu_check_prof.sh TAG CONFIG kernel_regex...
cd "$GRAFT_REPO_ROOT"
TAG=$1; C=$2; shift 2
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
mkdir -p /tmp/prof gpurun_out/prof_sum
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/prof/${C}_$k -f \
    python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$C $k rc=$?"
  python tools/ncu_summary.py full /tmp/prof/${C}_$k.ncu-rep gpurun_out/prof_sum/${TAG}_ncu_${C}_$k > /dev/null 2>&1
done
ls gpurun_out/prof_sum | tail -5
