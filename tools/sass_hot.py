#!/usr/bin/env python3
"""Per-region summary of an ncu source page (--page source --csv --print-source sass):
regions split at barriers (BAR), per region the executed instruction mix, the
warp-stall samples by reason, and shared-memory excess wavefronts (bank conflicts).

    ncu -i REP --page source --csv --launch-count 1 --print-source sass > x.csv
    python tools/sass_hot.py x.csv
"""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[i]
    recs = [dict(zip(hdr, r)) for r in rows[i + 1:] if len(r) == len(hdr)]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    regions = []
    cur = None
    for r in recs:
        src = r["Source"].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        if cur is None or op.startswith("BAR") and not op.startswith("BAR.ARV"):
            cur = {"start": r["Address"], "first": src[:60], "ops": collections.Counter(),
                   "exec": 0, "samples": collections.Counter(), "excess": 0, "wav": 0, "n": 0}
            regions.append(cur)
        ex = int(r["Instructions Executed"] or 0)
        cur["ops"][op.split(".")[0]] += ex
        cur["exec"] += ex
        cur["n"] += 1
        for c in stall_cols:
            v = r.get(c) or "0"
            cur["samples"][c[6:]] += int(v) if v.isdigit() else 0
        for key, col in (("excess", "L1 Wavefronts Shared Excessive"), ("wav", "L1 Wavefronts Shared")):
            v = r.get(col) or "0"
            cur[key] += int(v) if v.isdigit() else 0
    tot_s = sum(sum(g["samples"].values()) for g in regions) or 1
    tot_e = sum(g["exec"] for g in regions) or 1
    for g in regions:
        s = sum(g["samples"].values())
        if s < 0.005 * tot_s and g["exec"] < 0.005 * tot_e:
            continue
        top = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in g["samples"].most_common(5) if v)
        mix = ", ".join(f"{k} {v / max(g['exec'], 1) * 100:.0f}%" for k, v in g["ops"].most_common(6))
        print(f"{g['start']} n={g['n']:4d} samples {100 * s / tot_s:5.1f}% exec {100 * g['exec'] / tot_e:5.1f}%"
              f" smem-excess {g['excess']}/{g['wav']} | {g['first']}")
        print(f"      stalls: {top}")
        print(f"      mix:    {mix}")


if __name__ == "__main__":
    main(sys.argv[1])
