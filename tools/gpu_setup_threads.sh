# setup-CTA size variants: parity tests per variant, setup kernel time (launch list), frame rate
for t in 256 512 1024; do
  VR_LIB=build_variants/st$t.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
  VR_LIB=build_variants/st$t.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'vis_setup' --csv \
    --log-file gpurun_out/st_$t.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python - $t <<'PY'
import csv, sys
rows=[r for r in csv.reader(open(f"gpurun_out/st_{sys.argv[1]}.csv")) if len(r) > 10]
h=rows[0]; v=h.index("Metric Value"); x=[float(r[v].replace(",", "")) / 1e3 for r in rows[1:]]
print("setup threads", sys.argv[1], "vis_setup us", round(sum(x)/len(x), 1))
PY
done
CONFIGS="c3 c4" bash tools/variants.sh build_variants/st1024.so build_variants/st256.so build_variants/st512.so build_variants/st1024.so build_variants/st256.so build_variants/st512.so
