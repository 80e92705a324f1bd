# Round-end evidence on one B200 (run under gpurun): pytest -m gpu, smoke, default bench, ncu launch list +
# --set full captures (scripts/profile_r02.sh).  TAG names the outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG:-r02f}_smi.txt 2>&1
T0=$(date +%s)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG:-r02f}_pytest_gpu.txt 2>&1
echo "pytest rc=$? s=$(( $(date +%s) - T0 ))" | tee -a gpurun_out/${TAG:-r02f}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r02f}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG:-r02f}_bench.json 2> gpurun_out/${TAG:-r02f}_bench.err; echo "bench rc=$?"
TAG=${TAG:-r02f} bash scripts/profile_r02.sh > gpurun_out/${TAG:-r02f}_profile.log 2>&1; echo "profile rc=$?"
tail -3 gpurun_out/${TAG:-r02f}_pytest_gpu.txt
