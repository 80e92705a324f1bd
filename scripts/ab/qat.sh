set -u
mkdir -p gpurun_out
timeout 900 python bench.py --model reduced --mlp nvfp4 --train-seconds 60 --steady-seconds 0 > gpurun_out/r02qat_nvfp4.json 2> gpurun_out/r02qat_nvfp4.err; echo "nvfp4 qat rc=$?"
tail -5 gpurun_out/r02qat_nvfp4.err
