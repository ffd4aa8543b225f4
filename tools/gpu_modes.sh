cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for m in "classification=pre" "classification=preintegrated" "mode=isosurface"; do
  extra=""; [ "$m" = "mode=isosurface" ] && extra="--set isovalue=600"
  timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --set $m $extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $m', round(d['value'],1), d['samples_taken'], d['interpolated_samples'])"
done
