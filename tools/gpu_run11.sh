set -x
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -4
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_27b.json 2> gpurun_out/bench_27b.err; cat gpurun_out/bench_27b.json; tail -3 gpurun_out/bench_27b.err
timeout 900 python bench.py --config xl --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_xl5.json 2> gpurun_out/bench_xl5.err; cat gpurun_out/bench_xl5.json; tail -3 gpurun_out/bench_xl5.err
