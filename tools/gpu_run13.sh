set -x
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_27b_b.json 2> gpurun_out/bench_27b_b.err; cat gpurun_out/bench_27b_b.json; tail -3 gpurun_out/bench_27b_b.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 300 -c 3 -o gpurun_out/prof_step_gemm2 $CMD > gpurun_out/ncu13.log 2>&1; echo ncu rc=$?
