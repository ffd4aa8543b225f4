# Round-end measurement: tests, smoke, every bench line, the reference arm.
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r02}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
rm -f gpurun_out/bench_$TAG.jsonl
timeout 900 python bench.py >> gpurun_out/bench_$TAG.jsonl 2>> gpurun_out/bench_$TAG.err; echo "default rc=$?"
for c in c1 c2 c3soft c3stress c3pre c3preint c3iso c4 c5 k4; do
  st=20; [ "$c" = c5 ] && st=3; [ "$c" = c3stress ] && st=10
  timeout 900 python bench.py --config $c --steps $st --warmup 3 >> gpurun_out/bench_$TAG.jsonl 2>> gpurun_out/bench_$TAG.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/bench_$TAG.jsonl 2>> gpurun_out/bench_$TAG.err; echo "ref rc=$?"
python - "$TAG" <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_{sys.argv[1]}.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    r = d.get("roofline") or {}
    print(d.get("impl", "ours"), d["config"]["workload"], round(d["value"], 2), "e2e", round(e.get("value", 0) or 0, 1),
          "frac", round(r.get("frac", 0) or 0, 3), "cpu", round(cpu.get("value", 0) or 0, 3), (d.get("clocks") or {}).get("sm_mhz"))
PY
