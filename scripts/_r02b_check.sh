set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02b_smi.txt 2>&1
T0=$(date +%s)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_pytest_gpu.txt 2>&1
echo "pytest rc=$? s=$(( $(date +%s) - T0 ))" | tee -a gpurun_out/r02b_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02b_bench.json
tail -3 gpurun_out/r02b_pytest_gpu.txt
