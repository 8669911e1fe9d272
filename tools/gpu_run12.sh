set -x
nvidia-smi --query-gpu=index,name --format=csv
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -8
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_27b_n2.json 2> gpurun_out/bench_27b_n2.err; cat gpurun_out/bench_27b_n2.json; tail -5 gpurun_out/bench_27b_n2.err
