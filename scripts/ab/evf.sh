set -u
for rep in 1 2 3; do
 for v in base evf; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm 2>&1 | tail -1
 done
done
