#!/usr/bin/env bash
# compute-sanitizer over every libtang kernel (small batches; run on the B200 box under gpurun)
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-r02}
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_driver.py \
      > "$OUT/${TAG}_sanitize_$tool.txt" 2>&1
  echo "$tool rc=$?" >> "$OUT/${TAG}_sanitize_summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Error|Warning)|SANITIZE_DRIVER_DONE" "$OUT/${TAG}_sanitize_$tool.txt" | tail -4 >> "$OUT/${TAG}_sanitize_summary.txt"
done
cat "$OUT/${TAG}_sanitize_summary.txt"
