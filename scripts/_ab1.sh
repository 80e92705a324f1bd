set -u
mkdir -p gpurun_out
bash scripts/ab_micro.sh r02ab1 "base nobias nobias_nohld" "--mlp bf16 --N 512 --B 6"
cat gpurun_out/r02ab1_ab.txt
