set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02n_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02n_pytest.txt; tail -3 gpurun_out/r02n_pytest.txt
for v in base f8prev; do
 for cfg in "--N 512 --B 6" "--N 256 --B 2"; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v fp8 $cfg: " >> gpurun_out/r02n_ab.txt
  timeout 300 python scripts/mlp_micro.py --mlp fp8 $cfg --iters 10 2>&1 | tail -1 >> gpurun_out/r02n_ab.txt
 done
done
unset TANG_LIB
for k in auto wide; do echo -n "base bf16 $k: " >> gpurun_out/r02n_ab.txt; timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $k --iters 10 2>&1 | tail -1 >> gpurun_out/r02n_ab.txt; done
cat gpurun_out/r02n_ab.txt
