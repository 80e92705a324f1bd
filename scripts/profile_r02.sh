#!/usr/bin/env bash
# ncu evidence for the default bench workload (run on the B200 box): launch list of a short bench,
# one --set full capture of the MLP kernel (2SM, the shipped AUTO variant) and of the search kernels
# in the bench's own launch configuration (--cache-control none: tables warm in L2 as in the bench).
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-r02s}
mkdir -p "$OUT"
B="python bench.py --steps 3 --warmup 3 --steady-seconds 0 --no-cpu-baseline --p99-batches 10"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'mlp_tc|mlp_f8|probe|fallback|encode|apply_delta' \
    --csv --log-file "$OUT/${TAG}_launches.csv" $B > "$OUT/${TAG}_launches.out" 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:'mlp_tc_kernel' -s 4 -c 1 \
    -o "$OUT/${TAG}_mlp" $B > "$OUT/${TAG}_mlp.out" 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:'probe_kernel|probe_long_kernel|probe_finalize_kernel|fallback_kernel' -s 12 -c 4 \
    -o "$OUT/${TAG}_search" $B > "$OUT/${TAG}_search.out" 2>&1
for f in mlp search; do ncu -i "$OUT/${TAG}_$f.ncu-rep" --page raw --csv > "$OUT/${TAG}_${f}_raw.csv" 2>/dev/null; done
ls -la "$OUT" | grep "$TAG"
