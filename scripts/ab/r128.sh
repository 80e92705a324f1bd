set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/r02g_pytest.txt 2>&1; echo "guard pytest rc=$?"; tail -1 gpurun_out/r02g_pytest.txt
TANG_LIB=$PWD/variants/libtang_r128.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02r128_pytest.txt 2>&1; echo "r128 pytest rc=$?"; tail -1 gpurun_out/r02r128_pytest.txt
for rep in 1 2; do
 for v in base r128; do
  for k in single 2sm; do
   if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
   echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel $k 2>&1 | tail -1
  done
 done
 unset TANG_LIB; echo -n "base512: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm 2>&1 | tail -1
done | tee gpurun_out/r02r128_micro.txt
