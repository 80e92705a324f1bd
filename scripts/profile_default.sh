#!/usr/bin/env bash
# Run on the B200 box (under gpurun): default-workload evidence -- launch list of the bench command,
# one `ncu --set full` capture of the bf16 MLP kernel (a 1M-packet launch of scripts/mlp_micro.py) and
# the kernel's clock64 phase trace.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01h}
mkdir -p "$OUT"
CMD="python bench.py --steps 3 --warmup 1 --train-seconds 20 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'mlp_tc|probe|fallback_kernel|encode_kernel|apply_delta' \
    --csv --log-file "$OUT/${TAG}_launches.csv" $CMD > "$OUT/${TAG}_launches.out" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'mlp_tc_kernel' -s 2 -c 1 \
    -o "$OUT/${TAG}_mlp" python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --iters 2 > "$OUT/${TAG}_mlp.out" 2>&1
timeout 300 python scripts/mlp_trace.py > "$OUT/${TAG}_trace.txt" 2>&1
ls -la "$OUT"
