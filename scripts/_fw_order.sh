set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02fwo_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02fwo_pytest.txt
timeout 900 python bench.py --workload fw-512k --train-seconds 60 --steady-seconds 0 > gpurun_out/r02fwo_fw512k.json 2> gpurun_out/r02fwo_fw512k.err; echo "fw rc=$?"
timeout 900 python bench.py --workload fw-512k --train-seconds 60 --steady-seconds 0 --mode strict > gpurun_out/r02fwo_fw512k_strict.json 2> gpurun_out/r02fwo_fw512k_strict.err; echo "fw strict rc=$?"
