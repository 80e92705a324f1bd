set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k 2sm4 > gpurun_out/r02ab4_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02ab4_pytest.txt
for k in 2sm 2sm4; do bash scripts/ab_micro.sh r02ab4_$k "base noepi" "--mlp bf16 --N 512 --B 6 --kernel $k"; cat gpurun_out/r02ab4_${k}_ab.txt; done
timeout 200 python scripts/mlp_trace.py 2sm4 > gpurun_out/r02ab4_trace_2sm4.txt 2>&1
TANG_LIB=$PWD/variants/libtang_noepi.so timeout 200 python scripts/mlp_trace.py 2sm4 > gpurun_out/r02ab4_trace_noepi_2sm4.txt 2>&1
