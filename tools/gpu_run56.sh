# after the attention / dgrad-raster tuning: kernel tests, default bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -2
timeout 1500 python bench.py --steps 4 --warmup 3 > gpurun_out/bench56.json 2> gpurun_out/bench56.err; tail -2 gpurun_out/bench56.err
python -c "
import json
d=json.loads(open('gpurun_out/bench56.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], d['swap_hidden_pct'], d['compute_busy_pct'], d['step_roofline']['frac'], d['roofline']['achieved'], d['clocks'], d['cpu_baseline']['value'])
"
