# host update placement: GPU parity (oracle, swapped == resident with the CPU AdamW), regression of the step tests, 2.7B bench with 4 rounds per update
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_update.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -15
timeout 1500 python bench.py --steps 8 --warmup 4 --no-cpu-baseline --grad-rounds 4 --trace-out gpurun_out/trace46.txt > gpurun_out/bench46.json 2> gpurun_out/bench46.err; tail -3 gpurun_out/bench46.err
python -c "
import json
d=json.loads(open('gpurun_out/bench46.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], c['C'], c['act_policy'], c['n_recompute'], c['sub_models'], d['swap_hidden_pct'], d['compute_busy_pct'], d['h2d_GBs'], d['d2h_GBs'], d['step_roofline'], d['clocks'], d.get('host_link'))
"
