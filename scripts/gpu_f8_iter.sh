set -x
mkdir -p gpurun_out
T=$1
timeout 600 python -m pytest tests/test_gpu_fp8.py -q > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
for nb in "256 2" "256 4" "128 2"; do set -- $nb; timeout 120 python scripts/mlp_micro.py --mlp fp8 --N $1 --B $2 >> gpurun_out/${T}_micro.txt 2>&1; done
timeout 120 python scripts/mlp_trace_dual.py > gpurun_out/${T}_trace.txt 2>&1
