set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/gemm_perf.py 2>&1 | tail -14
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops 899 > gpurun_out/bench36.json 2> gpurun_out/bench36.err; tail -2 gpurun_out/bench36.err
python -c "
import json
d=json.load(open('gpurun_out/bench36.json')); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])
for r in d['roofline']['by_shape']: print(r)
"
