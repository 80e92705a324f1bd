#!/usr/bin/env python
"""Summarise ncu captures (run here, no GPU): launch-list shares and the key metrics of a
`--set full` report, written as JSON + Markdown under profiles/."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg",
]


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        import re
        m = re.search(r"(\w+_kernel)", r[ki])
        name = m.group(1) if m else r[ki][:40]
        agg[name][0] += float(r[vi].replace(",", ""))
        agg[name][1] += 1
    tot = sum(v[0] for v in agg.values())
    return {k: {"launches": v[1], "total_ns": v[0], "share": v[0] / tot} for k, v in agg.items()}


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for i, h in enumerate(hdr):
            if h in KEYS or any(h.startswith(k) for k in ("sm__pipe_tensor", "sm__inst_executed_pipe_tc")):
                d[h] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    tag = sys.argv[1]
    base = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    summ = {"launches": launches(f"{base}/{tag}_launches.csv")}
    for k in ("mlp", "search"):
        try:
            summ[k] = report(f"{base}/{tag}_{k}.ncu-rep")
        except Exception as e:
            summ[k] = str(e)
    print(json.dumps(summ, indent=1))
