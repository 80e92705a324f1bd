set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -m gpu -s > gpurun_out/r02f4_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02f4_pytest.txt
tail -2 gpurun_out/r02f4_pytest.txt
timeout 900 python bench.py --model reduced --mlp nvfp4 --train-seconds 60 > gpurun_out/r02ev_reduced_nvfp4.json 2> gpurun_out/r02ev_reduced_nvfp4.err; echo "bench nvfp4 rc=$?"
timeout 900 python bench.py --model reduced --mlp fp8 --train-seconds 60 --steady-seconds 0 > gpurun_out/r02ev_reduced_fp8_b.json 2> gpurun_out/r02ev_reduced_fp8_b.err; echo "bench fp8 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_f4_kernel -s 2 -c 1 -o gpurun_out/r02f4_ncu_v2 python scripts/mlp_micro.py --mlp nvfp4 --N 256 --B 2 --n 1048576 --iters 2 > gpurun_out/r02f4_ncu_v2.out 2>&1; echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f4_launches.csv python bench.py --model reduced --mlp nvfp4 --train-seconds 5 --steps 2 --warmup 1 --steady-seconds 0 --p99-batches 0 > /dev/null 2>&1; echo "launches rc=$?"
