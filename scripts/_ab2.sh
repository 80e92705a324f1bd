set -u
mkdir -p gpurun_out
bash scripts/ab_micro.sh r02ab2 "base noepi" "--mlp bf16 --N 512 --B 6"
cat gpurun_out/r02ab2_ab.txt
timeout 200 python scripts/mlp_trace.py 2sm > gpurun_out/r02ab2_trace_base.txt 2>&1
TANG_LIB=$PWD/variants/libtang_noepi.so timeout 200 python scripts/mlp_trace.py 2sm > gpurun_out/r02ab2_trace_noepi.txt 2>&1
