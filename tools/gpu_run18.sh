set -x
mkdir -p gpurun_out
timeout 120 ./tools/tmem_bw | grep mma
timeout 60 python tools/attn_one.py 1 512 2 128; timeout 60 python tools/attn_one.py 1 300 3 80
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/attn_perf.py 2>&1 | tail -5
timeout 300 python tools/gemm_perf.py 2>&1 | tail -14
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_27b_e.json 2> gpurun_out/bench_27b_e.err; cat gpurun_out/bench_27b_e.json; tail -3 gpurun_out/bench_27b_e.err
