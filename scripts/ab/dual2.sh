set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02dual2_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02dual2_pytest.txt
timeout 900 python bench.py --model reduced --train-seconds 60 --steady-seconds 0 > gpurun_out/r02dual2_reduced_bf16.json 2> gpurun_out/r02dual2_reduced_bf16.err; echo "bench rc=$?"
