set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_determinism.py -q > gpurun_out/r02h_determinism.txt 2>&1; echo "determinism rc=$?"; tail -3 gpurun_out/r02h_determinism.txt
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/r02h_$tag.json 2> gpurun_out/r02h_$tag.err; echo "$tag rc=$?"; }
run strict --mode strict --steady-seconds 0
run fp8_paper --mlp fp8 --train-seconds 60 --steady-seconds 0
run reduced_fp8 --model reduced --mlp fp8 --train-seconds 60 --steady-seconds 0
run reduced_bf16 --model reduced --train-seconds 60 --steady-seconds 0
run fw512k --workload fw-512k --train-seconds 60 --steady-seconds 0
run ipc512k --workload ipc-512k --train-seconds 60 --steady-seconds 0
