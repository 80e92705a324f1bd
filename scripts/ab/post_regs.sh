set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02pr_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02pr_pytest.txt
timeout 600 python bench.py --model reduced --steady-seconds 0 > gpurun_out/r02pr_reduced_bf16.json 2> gpurun_out/r02pr_reduced_bf16.err; echo "bf16 rc=$?"
timeout 900 python bench.py --model reduced --mlp nvfp4 --train-seconds 60 --steady-seconds 0 > gpurun_out/r02pr_reduced_nvfp4.json 2> gpurun_out/r02pr_reduced_nvfp4.err; echo "nvfp4 rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02pr_smoke.txt 2>&1; echo "smoke rc=$?"
