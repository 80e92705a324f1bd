#!/usr/bin/env python
"""Per-source-line warp-stall breakdown of one kernel from an ncu report (cuda,sass source page).
usage: ncu_lines.py REPORT [lo hi]  -- prints lines sorted by samples, with top stall reasons."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10 ** 9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: defaultdict(float))
text = {}
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ln = int(r[0])
    text[ln] = r[1]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h or h == "Warp Stall Sampling (All Samples)" \
                or h == "Instructions Executed":
            try:
                agg[ln][h] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
print(f"total samples {tot:.0f}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:40]:
    if not lo <= ln <= hi:
        continue
    s = v["Warp Stall Sampling (All Samples)"]
    if s == 0:
        continue
    st = sorted(((k[6:], x) for k, x in v.items() if k.startswith("stall_")), key=lambda kx: -kx[1])[:3]
    print(f"{ln:5d} {100 * s / tot:5.1f}% inst {v['Instructions Executed']:9.0f} "
          + " ".join(f"{k}:{100 * x / max(s, 1):.0f}%" for k, x in st) + " | " + text.get(ln, "")[:70].strip())
