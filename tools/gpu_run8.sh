set -x
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_xl3.json 2> gpurun_out/bench_xl3.err; cat gpurun_out/bench_xl3.json; tail -3 gpurun_out/bench_xl3.err
