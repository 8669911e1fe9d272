# round-1 re-entry check: full GPU suite, GEMM shapes serial, default bench (profiled plan, cpu baseline), reference arm
set -x
mkdir -p gpurun_out
free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; nproc
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/gemm_perf.py 2>&1 | tail -14
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench37.json 2> gpurun_out/bench37.err; tail -3 gpurun_out/bench37.err
python -c "
import json
d=json.load(open('gpurun_out/bench37.json')); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['step_roofline'], d['swap_hidden_pct'], d['clocks'], d['cpu_baseline'])
for r in d['roofline']['by_shape']: print(r)
"
