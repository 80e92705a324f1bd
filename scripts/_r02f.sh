set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02f_smi.txt 2>&1
T0=$(date +%s)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02f_pytest_gpu.txt 2>&1
echo "pytest rc=$? s=$(( $(date +%s) - T0 ))" | tee -a gpurun_out/r02f_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
TAG=r02f bash scripts/profile_r02.sh > gpurun_out/r02f_profile.log 2>&1; echo "profile rc=$?"
tail -3 gpurun_out/r02f_pytest_gpu.txt
