#!/usr/bin/env python
"""Summarise the round-2 ncu captures of the default bench workload (run here, no GPU):
profiles/<tag>_ncu_summary.json (key metrics per kernel) and the per-launch traffic that
bench.py's roofline objects read (profiles/ncu_traffic.json)."""
import csv
import json
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r02s"
BASE = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "lts__t_requests.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    return [{h: (v, u) for h, v, u in zip(hdr, row, units)} for row in r[2:]]


def val(d, k):
    v, u = d[k]
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


summ = {"tag": TAG, "kernels": []}
traffic = json.load(open("profiles/ncu_traffic.json"))
for f in ("mlp", "search"):
    for d in rows(f"{BASE}/{TAG}_{f}_raw.csv"):
        name = d["Kernel Name"][0].split("(")[0].split("::")[-1]
        e = {"kernel": name}
        for k in KEYS:
            if k in d:
                e[k] = f"{d[k][0]} {d[k][1]}".strip()
        summ["kernels"].append(e)
        packets = 4194304                      # bench batch (one launch per step)
        t = val(d, "gpu__time_duration.sum")
        dram = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
        lts = float(d["lts__t_sectors.sum"][0].replace(",", "")) * 32
        entry = {"dram_bytes_per_launch": dram, "lts_bytes_per_launch": lts, "packets_per_launch": packets,
                 "ncu_ms": t * 1e3,
                 "source": f"profiles/{TAG}_ncu_summary.json: {name} in `python bench.py --steps 3 --warmup 3` "
                           f"(ncu --set full --cache-control none, 4M-packet launch)"}
        if name.startswith("mlp_tc_kernel"):
            traffic["acl-512k/paper"] = dict(entry, source=entry["source"] + "; algorithmic = 64 MiB headers + "
                                             "6.3 MB bf16 weights + 16 MiB predictions")
        else:
            traffic.setdefault("acl-512k/paper/search", {})[name] = entry
json.dump(summ, open(f"profiles/{TAG}_ncu_summary.json", "w"), indent=1)
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(summ, indent=1)[:3000])
