set -u
mkdir -p gpurun_out
# control-warpgroup registers 32 -> 48 (tc2 dual-tile bf16 and the NVFP4 kernel): tests, then A/B
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_nvfp4.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02cr_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02cr_pytest.txt
for rep in 1 2 3; do
 for v in base oldtc2; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "bf16 dual $v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel dual 2>&1 | tail -1
 done
 for v in base oldf4; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "nvfp4 $v: "; timeout 200 python scripts/mlp_micro.py --mlp nvfp4 --N 256 --B 2 2>&1 | tail -1
 done
done
