#!/usr/bin/env bash
# Run on the B200 box (under gpurun): MLP micro-benchmark + phase traces of the bf16 variants.
# usage: TAG=r02a bash scripts/gpu_mlp_ab.sh [variants...]
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-r02}
mkdir -p "$OUT"
V=${*:-"single 2sm"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/${TAG}_smi.txt" 2>&1
for v in $V; do
  for rep in 1 2; do
    timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $v --iters 10 >> "$OUT/${TAG}_micro.txt" 2>&1
  done
  timeout 300 python scripts/mlp_trace.py $v > "$OUT/${TAG}_trace_$v.txt" 2>&1
done
cat "$OUT/${TAG}_micro.txt"
