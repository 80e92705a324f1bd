set -u
mkdir -p gpurun_out
for k in 2sm single; do
 for st in 4 5 6; do
  if [ $k = single ] && [ $st != 4 ]; then continue; fi
  echo -n "nobias S<=$st $k: " >> gpurun_out/r02i_ab.txt
  TANG_XSTAGES=$st TANG_LIB=$PWD/variants/libtang_nobias.so timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $k --iters 10 2>&1 | tail -1 >> gpurun_out/r02i_ab.txt
 done
 echo -n "base $k: " >> gpurun_out/r02i_ab.txt
 timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $k --iters 10 2>&1 | tail -1 >> gpurun_out/r02i_ab.txt
done
cat gpurun_out/r02i_ab.txt
