set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "timeline or stage2" > gpurun_out/r02y_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02y_pytest.txt; tail -2 gpurun_out/r02y_pytest.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 6 --warmup 3 --update-every 2 --no-cpu-baseline --p99-batches 100 > gpurun_out/r02y_torchrun_updates.json 2> gpurun_out/r02y_torchrun_updates.err; echo "torchrun rc=$?"; tail -c 600 gpurun_out/r02y_torchrun_updates.json
TAG=r02y bash scripts/profile_r02.sh > /dev/null 2>&1; ls gpurun_out | grep r02y
TAG=r02y bash scripts/sanitize.sh
