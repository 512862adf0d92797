#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/prof_bwd_r1e.ncu-rep --tag bwd_r01 \
        [--traffic-key hea20q:backward_pass]
    python tools/ncu_summary.py --launches gpurun_out/launches_r1a.csv --tag launches_r01

Writes profiles/<tag>.md (+ merges per-launch DRAM traffic into
profiles/ncu_traffic.json when --traffic-key is given).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(h, r):
    st = [(h[i], r[i]) for i in range(len(h))
          if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")]
    vals = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
            for k, v in st]
    tot = sum(v for _, v in vals) or 1.0
    return sorted(((k, v / tot * 100) for k, v in vals), key=lambda x: -x[1])[:8]


def summarise_rep(rep, tag, traffic_key=None):
    h, units, rows = raw_rows(rep)
    lines = [f"# ncu summary `{tag}`", "", f"source: `{os.path.basename(rep)}` "
             "(ncu --set full --clock-control none; per-launch replay, cold caches)", ""]
    traffic = []
    for n, r in enumerate(rows):
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines.append(f"## launch {n}: `{name[:110]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| {label} | {r[i]} | {units[i]} |")
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units[h.index("dram__bytes_read.sum")], 1)
        wr *= scale.get(units[h.index("dram__bytes_write.sum")], 1)
        traffic.append(rd + wr)
        lines.append("")
        lines.append("top stall reasons (% of samples): " +
                     ", ".join(f"{k} {v:.1f}" for k, v in stalls(h, r)))
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_key:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[traffic_key] = sum(traffic) / len(traffic)
        d[traffic_key + ":source"] = f"{tag} (mean dram read+write per launch over {len(traffic)} launches)"
        with open(p, "w") as f:
            json.dump(d, f, indent=1)
    print(f"profiles/{tag}.md ({len(rows)} launches)")


def summarise_launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    lines = [f"# ncu launch list `{tag}`", "",
             f"source: `{os.path.basename(path)}` (ncu --metrics gpu__time_duration.sum "
             "--clock-control none; serialised, cold-cache: compare shares, not absolutes)", "",
             "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:80]}` | {c} | {t / 1e6:.3f} | {t / c / 1e3:.1f} | {t / tot * 100:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"profiles/{tag}.md ({sum(v[0] for v in agg.values())} launches)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--traffic-key")
    a = ap.parse_args()
    if a.rep:
        summarise_rep(a.rep, a.tag, a.traffic_key)
    if a.launches:
        summarise_launches(a.launches, a.tag)
    return 0


if __name__ == "__main__":
    sys.exit(main())
