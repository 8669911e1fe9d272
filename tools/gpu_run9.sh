set -x
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/gemm_perf.py 2>&1 | tail -14
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_xl4.json 2> gpurun_out/bench_xl4.err; cat gpurun_out/bench_xl4.json; tail -3 gpurun_out/bench_xl4.err
