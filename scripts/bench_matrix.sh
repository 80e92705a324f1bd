# Secondary bench configurations (run under gpurun): FP8 / reduced / FW / IPC / 1M-rule updates / Zipf, plus
# the reference arm; outputs gpurun_out/r02ev_<config>.json.
set -u
mkdir -p gpurun_out
run() { tag=$1; shift; python bench.py "$@" > gpurun_out/${TAG:-r02ev}_$tag.json 2> gpurun_out/${TAG:-r02ev}_$tag.err; echo "$tag rc=$?"; }
run default
run fp8_paper --mlp fp8 --train-seconds 60
run reduced_fp8 --model reduced --mlp fp8 --train-seconds 60
run reduced_bf16 --model reduced --train-seconds 60
run fw512k --workload fw-512k --train-seconds 60 --steady-seconds 0
run ipc512k --workload ipc-512k --train-seconds 60 --steady-seconds 0
run acl1m_updates --workload acl-1m --update-every 2 --train-seconds 60 --steady-seconds 0
run acl100k_zipf --workload acl-100k-zipf --train-seconds 60 --steady-seconds 0
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/${TAG:-r02ev}_reference.json 2> gpurun_out/${TAG:-r02ev}_reference.err; echo "reference rc=$?"
run reduced_nvfp4 --model reduced --mlp nvfp4 --train-seconds 60 --steady-seconds 0
