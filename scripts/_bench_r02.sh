set -u
mkdir -p gpurun_out
T0=$(date +%s)
python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
echo "bench rc=$? seconds=$(( $(date +%s) - T0 ))"
tail -c 3000 gpurun_out/r02r_bench.json
bash scripts/sanitize.sh
