# host update placement with the CPU AdamW on its own stream: parity, then 2.7B at 4 and 1 rounds per update
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_update.py -x -q -m gpu 2>&1 | tail -3
for R in 4 1; do
timeout 1500 python bench.py --steps 8 --warmup 4 --no-cpu-baseline --grad-rounds $R --trace-out gpurun_out/trace47_R$R.txt > gpurun_out/bench47_R$R.json 2> gpurun_out/bench47_R$R.err; tail -2 gpurun_out/bench47_R$R.err
python -c "
import json
d=json.loads(open('gpurun_out/bench47_R$R.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], c['C'], c['act_policy'], c['n_recompute'], d['swap_hidden_pct'], d['compute_busy_pct'], d['h2d_GBs'], d['d2h_GBs'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d.get('host_link'))
"
done
