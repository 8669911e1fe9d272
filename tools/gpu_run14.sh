set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -6
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_27b_c.json 2> gpurun_out/bench_27b_c.err; cat gpurun_out/bench_27b_c.json; tail -3 gpurun_out/bench_27b_c.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_27b.csv $CMD > gpurun_out/ncu_launch14.log 2>&1
echo "launch rc=$?"
