set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -4
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops 899 > gpurun_out/bench31a.json 2> gpurun_out/bench31a.err; tail -2 gpurun_out/bench31a.err
ATOM_SIDE_WGRAD=0 timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops 899 > gpurun_out/bench31b.json 2> gpurun_out/bench31b.err; tail -2 gpurun_out/bench31b.err
python -c "
import json
for f in ('gpurun_out/bench31a.json','gpurun_out/bench31b.json'):
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])
"
