set -u
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 6 --warmup 3 --update-every 2 --no-cpu-baseline --p99-batches 100 --steady-seconds 0 > gpurun_out/r02k_torchrun_updates.json 2> gpurun_out/r02k_torchrun_updates.err; echo "torchrun rc=$?"
tail -c 400 gpurun_out/r02k_torchrun_updates.json
