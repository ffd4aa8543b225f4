cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/san
python tools/sanitize_smoke.py > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?"
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/san/$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san/$t.log
done
for m in "classification=pre" "classification=preintegrated" "mode=isosurface"; do
  extra=""; [ "$m" = "mode=isosurface" ] && extra="--set isovalue=600"
  timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --set $m $extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $m', round(d['value'],1), d['samples_taken'])"
done
timeout 300 python bench.py --config k4 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('k4', round(d['ms_per_step'],4), round(r['kernel_ms'],4), 'ms', round(r['frac'],3), 'balls', round(r['balls_ms'],4))"
