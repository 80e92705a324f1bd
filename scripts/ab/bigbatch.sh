set -u
mkdir -p gpurun_out
for m in fp8 bf16; do
  timeout 900 python bench.py --model reduced --mlp $m --train-seconds 30 --batch 16777216 --steady-seconds 0 --p99-batches 200 --no-cpu-baseline > gpurun_out/r02bb_$m.json 2> gpurun_out/r02bb_$m.err; echo "$m rc=$?"
done
