# re-entry confirmation (restored container) on one B200: build, GPU suite, smoke, default bench, reference arm
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1500 python bench.py > gpurun_out/bench63.json 2> gpurun_out/bench63.err; tail -2 gpurun_out/bench63.err
python -c "
import json
d=json.loads(open('gpurun_out/bench63.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], d['swap_hidden_pct'], d['step_roofline']['frac'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['cpu_baseline'])
"
timeout 1500 python bench.py --impl reference > gpurun_out/bench63_ref.json 2> gpurun_out/bench63_ref.err; cut -c1-300 gpurun_out/bench63_ref.json
