set -u
mkdir -p gpurun_out
for rep in 1 2; do
 for v in base ts_noepi ts_nosts; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel ts 2>&1 | tail -1
 done
done | tee gpurun_out/r02ts8_micro.txt
export TANG_LIB=$PWD/variants/libtang_ts_noepi.so; timeout 300 python scripts/mlp_trace_ts.py > gpurun_out/r02ts8_trace_noepi.txt 2>&1
export TANG_LIB=$PWD/variants/libtang_ts_nosts.so; timeout 300 python scripts/mlp_trace_ts.py > gpurun_out/r02ts8_trace_nosts.txt 2>&1
