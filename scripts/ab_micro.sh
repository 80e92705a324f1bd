#!/usr/bin/env bash
# A/B of MLP kernel variants (run on the B200 box): scripts/ab_micro.sh TAG "base v3 v5" "--mlp bf16 --N 512 --B 6"
T=$1; VARS=$2; ARGS=$3
mkdir -p gpurun_out
for rep in 1 2; do
for v in $VARS; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: " >> gpurun_out/${T}_ab.txt
  timeout 200 python scripts/mlp_micro.py $ARGS 2>&1 | tail -1 >> gpurun_out/${T}_ab.txt
done
done
