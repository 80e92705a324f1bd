set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02final_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02final_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02final_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02final_smoke.txt
