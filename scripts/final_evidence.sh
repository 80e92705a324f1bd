# Final-state evidence (run under gpurun): gpu_evidence.sh (pytest -m gpu, smoke, default bench, ncu) plus
# the reduced-model bf16 line (dual-tile kernel).
set -u
TAG=${TAG:-r02z} bash scripts/gpu_evidence.sh
timeout 900 python bench.py --model reduced --train-seconds 60 --steady-seconds 0 > gpurun_out/${TAG:-r02z}_reduced_bf16.json 2> gpurun_out/${TAG:-r02z}_reduced_bf16.err; echo "reduced bf16 rc=$?"
