set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py -q -x -k "dual" > gpurun_out/r02dual_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02dual_pytest.txt
for rep in 1 2; do for k in single dual; do timeout 200 python scripts/mlp_micro.py --mlp bf16 --N 256 --B 2 --kernel $k 2>&1 | tail -1; done; done | tee gpurun_out/r02dual_micro.txt
