set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/gemm_perf.py 2>&1 | tail -14
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench28.json 2> gpurun_out/bench28.err; cat gpurun_out/bench28.json; tail -3 gpurun_out/bench28.err
