#!/usr/bin/env python
"""Key metrics + stall breakdown + top stalled SASS lines of one ncu report (run here)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "dram__bytes_read.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in d: print(f"{k:80s} {d[k][0]} {d[k][1]}")
st = [(k, float(d[k][0].replace(',', ''))) for k in d if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued') and d[k][0] not in ('', 'n/a')]
tot = sum(x for _, x in st) or 1
for k, x in sorted(st, key=lambda t: -t[1])[:8]:
    print(f"  stall {x / tot * 100:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]; data = rows[2:]
si = hh.index("Warp Stall Sampling (All Samples)"); ii = hh.index("Instructions Executed")
tot = sum(float(r[si] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {float(r[si]) / tot * 100:5.1f}%  exec={r[ii]:>10}  {r[0][-5:]} {r[1].strip()[:80]}")
