set -u
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_tc.py -q -x -k "ts" > gpurun_out/r02ts4_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02ts4_pytest.txt
for rep in 1 2; do
 for v in base ts_gbias; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel ts 2>&1 | tail -1
 done
 unset TANG_LIB; echo -n "2sm: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm 2>&1 | tail -1
done | tee gpurun_out/r02ts4_micro.txt
unset TANG_LIB
timeout 300 python scripts/mlp_trace_ts.py > gpurun_out/r02ts4_trace.txt 2>&1
TANG_LIB=$PWD/variants/libtang_ts_gbias.so timeout 300 python scripts/mlp_trace_ts.py > gpurun_out/r02ts4_trace_gbias.txt 2>&1
