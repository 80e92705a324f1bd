set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/r02tw_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02tw_pytest.txt
for rep in 1 2; do for k in 2sm single wide; do timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel $k 2>&1 | tail -1; done; done | tee gpurun_out/r02tw_micro.txt
timeout 300 python scripts/mlp_trace.py 2sm > gpurun_out/r02tw_trace.txt 2>&1
