set -u
timeout 600 python -m pytest tests/test_c_abi_demo.py -q -s > gpurun_out/r02cdemo_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02cdemo_pytest.txt
