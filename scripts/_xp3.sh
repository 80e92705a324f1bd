set -u
mkdir -p gpurun_out
./scripts/l2_gather > gpurun_out/r02q_l2_gather.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc.py "tests/test_gpu_fullsize.py::test_512k_headline_trained_model_logits_and_rule_ids" "tests/test_gpu_fullsize.py::test_256k_long_churn_50_windows" -x -q -m gpu -s > gpurun_out/r02q_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02q_pytest.txt
tail -3 gpurun_out/r02q_pytest.txt; grep -E "headline|churn" gpurun_out/r02q_pytest.txt
for rep in 1 2; do for v in base wu; do
  if [ $v = base ]; then unset TANG_LIB; else export TANG_LIB=$PWD/variants/libtang_$v.so; fi
  echo -n "$v 2sm: " >> gpurun_out/r02q_ab.txt
  timeout 300 python scripts/mlp_micro.py --mlp bf16 --N 512 --B 6 --kernel 2sm --iters 10 2>&1 | tail -1 >> gpurun_out/r02q_ab.txt
done; done
unset TANG_LIB
timeout 300 python scripts/mlp_trace.py 2sm > gpurun_out/r02q_trace_2sm.txt 2>&1
cat gpurun_out/r02q_ab.txt gpurun_out/r02q_l2_gather.txt
