set -u
mkdir -p gpurun_out
for rb in 1048576 2097152 4194304; do
  timeout 600 python bench.py --ring-batch $rb --steady-seconds 0 --p99-batches 200 --no-cpu-baseline > gpurun_out/r02ring_$rb.json 2> gpurun_out/r02ring_$rb.err; echo "rb=$rb rc=$?"
done
