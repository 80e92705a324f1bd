set -u
mkdir -p gpurun_out
bash scripts/ab_micro.sh r02ab3 "noepi noepi6 noepi3" "--mlp bf16 --N 512 --B 6"
cat gpurun_out/r02ab3_ab.txt
TANG_LIB=$PWD/variants/libtang_noepi6.so timeout 200 python scripts/mlp_trace.py 2sm > gpurun_out/r02ab3_trace_noepi6.txt 2>&1
