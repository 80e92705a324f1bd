set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steady-seconds 60 --p99-batches 1000 --no-cpu-baseline > gpurun_out/r02_steady60.json 2> gpurun_out/r02_steady60.err; echo "rc=$?"
