set -u
mkdir -p gpurun_out
TANG_LIB=$PWD/variants/libtang_f8tail.so timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02f8tail_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02f8tail_pytest.txt
for rep in 1 2; do
 for v in base f8tail; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp fp8 --N 256 --B 2 2>&1 | tail -1
 done
done
