#!/usr/bin/env bash
# Kernel iteration on the B200 box: correctness gate, A/B micro vs variant libraries, phase traces.
# usage: TAG=r02c VARIANTS="base r01" KERNELS="single 2sm" TESTS="tests/test_gpu_tc.py" bash scripts/gpu_iter.sh
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-r02}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/${TAG}_smi.txt" 2>&1
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -x -q -m gpu > "$OUT/${TAG}_pytest.txt" 2>&1; echo "pytest rc=$?" >> "$OUT/${TAG}_pytest.txt"
  tail -3 "$OUT/${TAG}_pytest.txt"
fi
for k in ${KERNELS:-single}; do
  for rep in 1 2; do
    for v in ${VARIANTS:-base}; do
      if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
      echo -n "$v $k: " >> "$OUT/${TAG}_ab.txt"
      timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $k --iters 10 ${MICRO_ARGS:-} 2>&1 | tail -1 >> "$OUT/${TAG}_ab.txt"
    done
  done
  unset TANG_LIB
  if [ -z "${NOTRACE:-}" ]; then timeout 300 python scripts/mlp_trace.py $k > "$OUT/${TAG}_trace_$k.txt" 2>&1; fi
done
cat "$OUT/${TAG}_ab.txt"
