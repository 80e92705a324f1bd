#!/usr/bin/env bash
# MLP kernel variants of one build (run on the B200 box): scripts/ab_kernels.sh TAG "single 2sm wide" "--mlp bf16 --N 512 --B 6"
T=$1; KS=$2; ARGS=$3
mkdir -p gpurun_out
for rep in 1 2; do
for k in $KS; do
  echo -n "$k: " >> gpurun_out/${T}_kernels.txt
  timeout 200 python scripts/mlp_micro.py $ARGS --kernel $k 2>&1 | tail -1 >> gpurun_out/${T}_kernels.txt
done
done
