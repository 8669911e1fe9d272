# round 2, run 68 (4 GPUs): the final tree's 4-peer and 2-peer bench lines on one box (torchrun,
# weak scaling, live link probe)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi -L
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2_68_n4.json 2> gpurun_out/r2_68_n4.err; echo rc=$?
tail -c 400 gpurun_out/r2_68_n4.json
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_68_n2.json 2> gpurun_out/r2_68_n2.err; echo rc=$?
tail -c 400 gpurun_out/r2_68_n2.json
