set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -2
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops 899 > gpurun_out/bench32.json 2> gpurun_out/bench32.err; tail -2 gpurun_out/bench32.err
python -c "
import json
d=json.load(open('gpurun_out/bench32.json')); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])
"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 899"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 60 -c 4 -o gpurun_out/prof_gemm32 $CMD > gpurun_out/ncu32.log 2>&1; echo "full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:col_sums -s 40 -c 4 -o gpurun_out/prof_cs32 $CMD > gpurun_out/ncu32b.log 2>&1; echo "full rc=$?"
