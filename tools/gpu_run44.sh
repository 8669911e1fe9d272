# one-wave column sums: step parity tests, the column-sum kernels under ncu, default bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -3
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7"
timeout 900 ncu --set full --clock-control none -k regex:"col_sums" -c 4 -o gpurun_out/prof_cs44 $CMD > gpurun_out/ncu44.log 2>&1; echo "ncu rc=$?"
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench44.json 2> gpurun_out/bench44.err; tail -2 gpurun_out/bench44.err
python -c "
import json
d=json.loads(open('gpurun_out/bench44.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], c['C'], c['act_policy'], c['n_recompute'], d['swap_hidden_pct'], d['step_roofline']['frac'], d['roofline']['achieved'], d['clocks'])
"
