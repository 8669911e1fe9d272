set -x
mkdir -p gpurun_out
timeout 300 python tools/gemm_perf.py 2>&1 | tail -20
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -5
timeout 120 python tools/gemm_one.py 16384 10240 2560 0 0 512 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_gemm2 python tools/gemm_one.py 16384 10240 2560 0 0 512 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/prof_gemm1 python tools/gemm_one.py 16384 10240 2560 0 0 256 > gpurun_out/ncu1.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_xl2.json 2> gpurun_out/bench_xl2.err; cat gpurun_out/bench_xl2.json; tail -3 gpurun_out/bench_xl2.err
