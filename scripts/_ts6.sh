set -u
mkdir -p gpurun_out
export TANG_LIB=$PWD/variants/libtang_ts_noepi.so
for rep in 1 2; do echo -n "ts_noepi: "; timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel ts 2>&1 | tail -1; done | tee gpurun_out/r02ts6_micro.txt
timeout 300 python scripts/mlp_trace_ts.py > gpurun_out/r02ts6_trace_noepi.txt 2>&1
