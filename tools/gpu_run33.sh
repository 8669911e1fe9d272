set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_attention.py tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -2
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops 899 > gpurun_out/bench33.json 2> gpurun_out/bench33.err; tail -2 gpurun_out/bench33.err
python -c "
import json
d=json.load(open('gpurun_out/bench33.json')); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])
"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 899"
timeout 600 ncu --set full --clock-control none -k regex:col_sums -s 40 -c 4 -o gpurun_out/prof_cs33 $CMD > gpurun_out/ncu33b.log 2>&1; echo "full rc=$?"
