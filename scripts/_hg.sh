set -u
mkdir -p gpurun_out
for rep in 1 2; do
 for v in base half_grid; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm 2>&1 | tail -1
 done
done | tee gpurun_out/r02_half_grid.txt
export TANG_LIB=$PWD/variants/libtang_half_grid.so
timeout 200 python scripts/mlp_trace.py 2sm > gpurun_out/r02_half_grid_trace.txt 2>&1
