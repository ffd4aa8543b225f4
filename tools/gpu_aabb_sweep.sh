# AABB-fit grid size sweep (CTAs per SM): kernel time from the launch list, frame rate from bench
for n in 2 4 5 8 16; do
  VR_AABB_CTAS=$n timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'aabb|vis_setup' --csv \
    --log-file gpurun_out/aabb_$n.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python - $n <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open(f"gpurun_out/aabb_{sys.argv[1]}.csv")) if len(r) > 10]
h=rows[0]; k=h.index("Kernel Name"); v=h.index("Metric Value"); d=collections.defaultdict(list)
for r in rows[1:]: d[r[k][:20]].append(float(r[v].replace(",", "")) / 1e3)
print("ctas/sm", sys.argv[1], {a: round(sum(b)/len(b), 1) for a, b in d.items()})
PY
done
for n in 5 8 5 8; do VR_AABB_CTAS=$n timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas $n', round(d['value'],1), round(d['ms_per_step']-d['roofline']['kernel_ms'],4))"; done
