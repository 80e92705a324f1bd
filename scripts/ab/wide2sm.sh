set -u
mkdir -p gpurun_out
TANG_LIB=$PWD/variants/libtang_wide2sm.so timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "2sm" > gpurun_out/r02w2_pytest.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02w2_pytest.txt
for rep in 1 2; do
 for v in base wide2sm; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm 2>&1 | tail -1
 done
done
