set -u
mkdir -p gpurun_out
# dual-tile bf16 output layer, top-1 without logits: 32-column tree argmax in registers (base) vs
# per-column scan of 16-column loads (notree)
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -x -k "dual or determin or reduced" > gpurun_out/r02tree_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02tree_pytest.txt
for rep in 1 2 3; do
 for v in base notree; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "bf16 dual N256 $v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel dual 2>&1 | tail -1
 done
done
unset TANG_LIB
timeout 600 python bench.py --model reduced --steady-seconds 0 > gpurun_out/r02tree_reduced_bf16.json 2> gpurun_out/r02tree_reduced_bf16.err; echo "bench rc=$?"
