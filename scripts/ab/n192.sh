set -u
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "192" > gpurun_out/r02n192_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02n192_pytest.txt
