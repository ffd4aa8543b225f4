"""Group an ncu source page (cuda,sass csv) by source line / line range.

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [file:a-b ...]
"""
import csv
import sys
from collections import defaultdict


def load(path):
    agg = defaultdict(lambda: [0, 0, ""])
    cur_file = cur = None
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] in ("Function Name", "Line No"):
            continue
        if row[0].isdigit():
            cur = (cur_file, int(row[0]))
            try:
                agg[cur][0] += int(row[4])
                agg[cur][1] += int(row[7])
                agg[cur][2] = row[1].strip()[:80]
            except (ValueError, IndexError):
                pass
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    S = sum(v[0] for v in agg.values()) or 1
    I = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {S} instructions {I}")
    for spec in sys.argv[2:]:
        f, r = spec.split(":")
        a, b = (int(x) for x in r.split("-"))
        s = sum(v[0] for k, v in agg.items() if k[0] == f and a <= k[1] <= b)
        i = sum(v[1] for k, v in agg.items() if k[0] == f and a <= k[1] <= b)
        print(f"{spec:28s} samples {s / S:.3f} inst {i / I:.3f}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{k[0]}:{k[1]:5d} smp {v[0] / S:.3f} inst {v[1] / I:.3f}  {v[2]}")
