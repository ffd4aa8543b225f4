# per-kernel duration / instructions / fp64 pipe for library variants: bash tools/ncu_kernels.sh CONFIG lib1.so lib2.so
C=$1; shift
for lib in "$@"; do
  VR_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:raycast -c 4 --csv \
    python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncuk.csv 2>/dev/null
  python - "$lib" <<'PY'
import csv, sys
rows = list(csv.reader(open("gpurun_out/ncuk.csv")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h, rows = rows[hi], [r for r in rows[hi:] if len(r) == len(rows[hi])]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    print(sys.argv[1], r[ki].split("(")[0][-40:], r[mi], r[vi])
PY
done
