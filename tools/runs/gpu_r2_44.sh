# round 2, run 44 (2 GPUs): the final tree's multi-peer and elastic GPU tests, then the 2-peer bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi -L
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_elastic.py -v 2>&1 > gpurun_out/r2_44_multi.log; echo rc=$?
tail -15 gpurun_out/r2_44_multi.log
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_44_n2.json 2> gpurun_out/r2_44_n2.err; echo rc=$?
tail -c 600 gpurun_out/r2_44_n2.json
tail -3 gpurun_out/r2_44_n2.err
