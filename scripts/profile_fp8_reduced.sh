#!/usr/bin/env bash
# Run on the B200 box (under gpurun): reduced-model FP8 evidence -- bench lines (ring-slot sweep for
# the e2e leg), the launch list of the bench command, and one `ncu --set full` capture of the
# dual-tile MLP kernel (one 4M-packet launch of scripts/mlp_micro.py, the bench's launch size).
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01g}
mkdir -p "$OUT"
for rb in 262144 1048576; do
  timeout 600 python bench.py --model reduced --mlp fp8 --ring-batch $rb > "$OUT/${TAG}_bench_rb$rb.json" 2> "$OUT/${TAG}_bench_rb$rb.err"
done
CMD="python bench.py --model reduced --mlp fp8 --steps 3 --warmup 1 --train-seconds 20 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'mlp_f8|probe|fallback_kernel|encode_kernel|apply_delta' \
    --csv --log-file "$OUT/${TAG}_launches.csv" $CMD > "$OUT/${TAG}_launches.out" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'mlp_f8x2' -s 2 -c 1 \
    -o "$OUT/${TAG}_mlp_f8x2" python scripts/mlp_micro.py --mlp fp8 --N 256 --B 2 --iters 2 > "$OUT/${TAG}_mlp_f8x2.out" 2>&1
ls -la "$OUT"
