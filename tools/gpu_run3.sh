set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_xl.json 2> gpurun_out/bench_xl.err
tail -5 gpurun_out/bench_xl.err; cat gpurun_out/bench_xl.json
