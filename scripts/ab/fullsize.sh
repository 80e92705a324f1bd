set -u
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "512k_sampled" > gpurun_out/r02fs_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02fs_pytest.txt
