# the other BASELINE configs on one B200 with the current kernels: GPT-3 Small (per-layer sub-models), XL
set -x
mkdir -p gpurun_out
for CFG in small xl; do
timeout 1500 python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench48_$CFG.json 2> gpurun_out/bench48_$CFG.err; tail -2 gpurun_out/bench48_$CFG.err
python -c "
import json
d=json.loads(open('gpurun_out/bench48_$CFG.json').read().strip().splitlines()[-1]); c=d['config']
print('$CFG', d['value'], d['ms_per_step'], c['C'], c['act_policy'], c['sub_models'], d['swap_hidden_pct'], d['compute_busy_pct'], d['step_roofline']['frac'], d['roofline']['achieved'], d['clocks']['sm_mhz'])
"
done
