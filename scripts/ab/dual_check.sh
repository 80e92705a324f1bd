set -u
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -q -x > gpurun_out/r02dc_pytest.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02dc_pytest.txt
