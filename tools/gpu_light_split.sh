# per-kernel time with lighting on / off (launch list), c3 and c3soft
for c in c3 c3soft; do for l in true false; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raycast --csv \
    --log-file gpurun_out/split_${c}_$l.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --set lighting=$l > /dev/null 2>&1
  python - $c $l <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open(f"gpurun_out/split_{sys.argv[1]}_{sys.argv[2]}.csv")) if len(r) > 10]
h=rows[0]; k=h.index("Kernel Name"); v=h.index("Metric Value"); d=collections.defaultdict(list)
for r in rows[1:]: d[r[k][:30]].append(float(r[v].replace(",", "")) / 1e3)
print(sys.argv[1], "lighting", sys.argv[2], {a: round(sum(b)/len(b), 1) for a, b in d.items()})
PY
done; done
