#!/usr/bin/env bash
# Run on the B200 box (under gpurun): one `ncu --set full` capture per bf16 MLP variant (a 1M-packet
# launch of scripts/mlp_micro.py), raw metrics exported as CSV next to the report.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-r02}
mkdir -p "$OUT"
for v in ${*:-single 2sm}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'mlp_tc_kernel' -s 2 -c 1 \
      -o "$OUT/${TAG}_mlp_$v" python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --n 1048576 --iters 2 --kernel $v \
      > "$OUT/${TAG}_mlp_$v.out" 2>&1
  ncu -i "$OUT/${TAG}_mlp_$v.ncu-rep" --page raw --csv > "$OUT/${TAG}_mlp_${v}_raw.csv" 2>/dev/null
done
ls -la "$OUT"
