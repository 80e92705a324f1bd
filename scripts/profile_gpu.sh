#!/usr/bin/env bash
# Run on the B200 box (under gpurun): launch list of the bench command + one `ncu --set full`
# capture of each hot kernel.  Summaries are parsed here with scripts/ncu_summary.py.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p "$OUT"
CMD="python bench.py --steps 3 --warmup 1 --train-seconds ${TRAIN_S:-20} --no-cpu-baseline ${BENCH_ARGS:-}"
# 1) every launch of our kernels with its device time (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'mlp_tc|mlp_pair|mlp_ffma|probe_kernel|fallback_kernel|encode_kernel|apply_delta' \
    --csv --log-file "$OUT/${TAG}_launches.csv" $CMD > "$OUT/${TAG}_launches.out" 2>&1
# 2) full section set of the MLP kernel (one launch of the timed region)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'mlp_tc_kernel|mlp_pair_kernel' -s 6 -c 1 \
    -o "$OUT/${TAG}_mlp" $CMD > "$OUT/${TAG}_mlp.out" 2>&1
# 3) full section set of probe + fallback
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'probe_kernel|fallback_kernel' -s 12 -c 2 \
    -o "$OUT/${TAG}_search" $CMD > "$OUT/${TAG}_search.out" 2>&1
ls -la "$OUT"
