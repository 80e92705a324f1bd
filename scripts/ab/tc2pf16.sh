set -u
mkdir -p gpurun_out
# dual-tile bf16 epilogue: 16-column chunks with the next chunk's TMEM load in flight (base) vs
# 32-column load-then-wait chunks (nopf)
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py -q -x -k "dual or determin" > gpurun_out/r02pf_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02pf_pytest.txt
for rep in 1 2 3; do
 for v in base nopf; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "bf16 dual N256 $v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel dual 2>&1 | tail -1
  echo -n "bf16 dual N128 $v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 128 --B 2 --kernel dual 2>&1 | tail -1
 done
done
