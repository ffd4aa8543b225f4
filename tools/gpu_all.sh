# full GPU test suite + every bench config (short runs); results in gpurun_out/all_<tag>.jsonl
cd "$GRAFT_REPO_ROOT"
TAG=${1:-x}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
rm -f gpurun_out/all_$TAG.jsonl
for c in c3 c2 c1 c3soft c3stress c4 c5 k4; do
  st=20; [ "$c" = c5 ] && st=3
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline >> gpurun_out/all_$TAG.jsonl 2>> gpurun_out/all_$TAG.err
done
python - "$TAG" <<'PY'
import json, sys
for l in open(f"gpurun_out/all_{sys.argv[1]}.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    e = d.get("e2e") or {}
    print(d["config"]["workload"], round(d["value"], 1), "e2e", round(e.get("value", 0), 1), "frac", round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"])
PY
