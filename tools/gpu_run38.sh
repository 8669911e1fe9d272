# 4 peers (one per GPU, NCCL averaging) on GPT-3 2.7B, then 2 peers; host memory probe
set -x
mkdir -p gpurun_out
free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; nproc; nvidia-smi topo -m
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench38_n4.json 2> gpurun_out/bench38_n4.err; tail -5 gpurun_out/bench38_n4.err
cut -c1-1500 gpurun_out/bench38_n4.json
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench38_n2.json 2> gpurun_out/bench38_n2.err; tail -5 gpurun_out/bench38_n2.err
cut -c1-1500 gpurun_out/bench38_n2.json
