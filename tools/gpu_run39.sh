# host-link contention at 4 GPUs: copy probe at 1/2/4 ranks, then 4 peers with the last step's trace
set -x
mkdir -p gpurun_out
numactl -H 2>/dev/null | head -5; lscpu | grep -i "numa\|model name\|socket"
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/host_bw_probe.py
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/host_bw_probe.py 2>&1 | grep world
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 tools/host_bw_probe.py 2>&1 | grep world
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --steps 4 --warmup 3 --no-cpu-baseline --trace-out gpurun_out/trace39_n4.txt > gpurun_out/bench39_n4.json 2> gpurun_out/bench39_n4.err; tail -3 gpurun_out/bench39_n4.err
