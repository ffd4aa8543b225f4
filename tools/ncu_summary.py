"""Summarise ncu captures into profiles/ (runs here, no GPU).

    python tools/ncu_summary.py launches gpurun_out/launches_c3.csv profiles/r01_launches_c3.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r01_ncu_raycast_c3 [config]
    python tools/ncu_summary.py traffic c3 profiles/a.json profiles/b.json   # kernels of one frame

`full` writes <out>.md (metrics + top source lines) and <out>.json; with a
config name it also writes profiles/ncu_raycast_<config>.json, which
bench.py reads for roofline.traffic (dram bytes per launch).
"""

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

TIME_UNITS = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
              "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__inst_executed_op_global_ld.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(csv_path, out):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# Kernel launch list: `{Path(csv_path).name}`", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches:",
             "compare shares, not absolutes).", "",
             "| kernel | launches | mean us | total share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        name = k.split("(")[0].replace("vr::<unnamed>::", "")[:70]
        lines.append(f"| `{name}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, config=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2]
    vals = {}
    for i, name in enumerate(h):
        if name in METRICS or name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                vals[name] = float(v[i].replace(",", ""))
            except ValueError:
                vals[name] = v[i]
    kernel = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    units = {name: rows[1][i] for i, name in enumerate(h)}
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    samples, insts, text = defaultdict(int), defaultdict(int), {}
    cur_file = cur = None
    for row in csv.reader(src.splitlines()):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] in ("Function Name", "Line No"):
            continue
        if row[0].isdigit():
            cur = (cur_file, int(row[0]))
            text[cur] = row[1].strip()[:90]
        try:
            samples[cur] += int(row[4])
            insts[cur] += int(row[7])
        except (ValueError, IndexError):
            pass
    tot_s = sum(samples.values()) or 1
    tot_i = sum(insts.values()) or 1
    def scaled(name):
        x = vals.get(name)
        u = units.get(name, "")
        if isinstance(x, float) and u in ("Kbyte", "Mbyte", "Gbyte", "byte"):
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        if isinstance(x, float) and u in TIME_UNITS:
            return x * TIME_UNITS[u]
        return x
    dram = (scaled("dram__bytes_read.sum") or 0) + (scaled("dram__bytes_write.sum") or 0)
    summary = {"kernel": kernel, "report": Path(rep).name, "duration_s": scaled("gpu__time_duration.sum"),
               "dram_bytes_per_launch": dram,
               "metrics": {k: [vals[k], units.get(k, "")] for k in sorted(vals)},
               "top_lines": [[f"{k[0]}:{k[1]}", samples[k] / tot_s, insts[k] / tot_i, text.get(k, "")]
                             for k, _ in sorted(samples.items(), key=lambda x: -x[1])[:60]],
               "top_inst_lines": [[f"{k[0]}:{k[1]}", samples[k] / tot_s, insts[k] / tot_i, text.get(k, "")]
                                  for k, _ in sorted(insts.items(), key=lambda x: -x[1])[:80]]}
    Path(out + ".json").write_text(json.dumps(summary, indent=1))
    md = [f"# ncu --set full: `{kernel.split('(')[0]}`", "", f"report: `{Path(rep).name}` (gpurun_out, not committed)", "",
          "| metric | value | unit |", "|---|---:|---|"]
    for k in METRICS:
        if k in vals:
            md.append(f"| {k} | {vals[k]} | {units.get(k, '')} |")
    md += ["", "Warp-stall samples:", "", "| reason | samples |", "|---|---:|"]
    for k, x in sorted(((k, x) for k, x in vals.items() if k.startswith("smsp__pcsamp")), key=lambda t: -t[1]):
        if x:
            md.append(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {int(x)} |")
    md += ["", "Top source lines (share of stall samples / of executed instructions):", "",
           "| line | samples | instructions | source |", "|---|---:|---:|---|"]
    for loc, s_, i_, t in summary["top_lines"]:
        md.append(f"| {loc} | {s_:.3f} | {i_:.3f} | `{t}` |")
    Path(out + ".md").write_text("\n".join(md) + "\n")
    if config:
        Path(f"profiles/ncu_raycast_{config}.json").write_text(json.dumps(
            {"kernel": kernel, "dram_bytes_per_launch": dram, "source": Path(out + ".json").name}, indent=1))
    print("\n".join(md[:40]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "traffic":
        # kernels of one frame: DRAM bytes summed, utilisation duration-weighted
        parts = [json.loads(Path(p).read_text()) for p in sys.argv[3:]]

        def metric(p, name):
            m = p["metrics"].get(name)
            return float(m[0]) if m and isinstance(m[0], (int, float)) else None

        def seconds(p):
            m = p["metrics"].get("gpu__time_duration.sum")
            if m and isinstance(m[0], (int, float)) and m[1] in TIME_UNITS:
                return float(m[0]) * TIME_UNITS[m[1]]
            return p.get("duration_s") or 0.0

        for p in parts:
            p["duration_s"] = seconds(p)

        def weighted(name):
            num = den = 0.0
            for p in parts:
                v, d = metric(p, name), p.get("duration_s") or 0.0
                if v is not None:
                    num += v * d
                    den += d
            return num / den if den else None

        Path(f"profiles/ncu_raycast_{sys.argv[2]}.json").write_text(json.dumps(
            {"kernels": " + ".join(p["kernel"].split("(")[0] for p in parts),
             "dram_bytes_per_launch": sum(p["dram_bytes_per_launch"] for p in parts),
             "per_kernel": {p["kernel"].split("(")[0]: {
                 "dram_bytes": p["dram_bytes_per_launch"], "duration_s": p.get("duration_s"),
                 "issue_active_pct": metric(p, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "fp64_pipe_pct": metric(p, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                 "warps_active_pct": metric(p, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                 "l1_hit_pct": metric(p, "l1tex__t_sector_hit_rate.pct"),
                 "l1_bytes": metric(p, "l1tex__t_bytes.sum"), "l2_bytes": metric(p, "lts__t_bytes.sum")}
                 for p in parts},
             "issue_active_pct": weighted("smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "fp64_pipe_pct": weighted("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": weighted("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "l1_hit_pct": weighted("l1tex__t_sector_hit_rate.pct"),
             "l2_hit_pct": weighted("lts__t_sector_hit_rate.pct"),
             "source": [Path(p).name for p in sys.argv[3:]]}, indent=1))
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
