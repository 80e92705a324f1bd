set -u
mkdir -p gpurun_out
# FP8 dual-tile kernel: control-warpgroup registers 32 -> 64 (epilogue 112 -> 104): tests, then A/B
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02cr8_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02cr8_pytest.txt
for rep in 1 2 3; do
 for v in base oldf8; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "fp8 dual $v: "; timeout 200 python scripts/mlp_micro.py --mlp fp8 --N 256 --B 2 2>&1 | tail -1
 done
done
unset TANG_LIB
timeout 600 python bench.py --model reduced --mlp fp8 --steady-seconds 0 > gpurun_out/r02cr8_bench_reduced_fp8.json 2> gpurun_out/r02cr8_bench.err; echo "bench rc=$?"; cat gpurun_out/r02cr8_bench_reduced_fp8.json | head -c 600
