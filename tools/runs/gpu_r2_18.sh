# round 2, run 18 (4 GPUs): 4-peer bench (torchrun, weak scaling, live link probe)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --steps 8 --warmup 3 > gpurun_out/r2_18_n4.json 2> gpurun_out/r2_18_n4.err; echo rc=$?
tail -c 1500 gpurun_out/r2_18_n4.json
tail -5 gpurun_out/r2_18_n4.err
