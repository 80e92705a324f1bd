set -u
mkdir -p gpurun_out
TANG_LIB=$PWD/variants/libtang_tc2max.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py -q -x -k "dual" > gpurun_out/r02mx_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02mx_pytest.txt
for rep in 1 2; do
 for v in base tc2max; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel dual 2>&1 | tail -1
 done
done
