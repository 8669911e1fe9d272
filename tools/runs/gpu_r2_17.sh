# round 2, run 17 (2 GPUs): 2-peer bench (torchrun, weak scaling, live link probe)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_17_n2.json 2> gpurun_out/r2_17_n2.err; echo rc=$?
tail -c 1500 gpurun_out/r2_17_n2.json
tail -5 gpurun_out/r2_17_n2.err
