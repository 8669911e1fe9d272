# re-entry confirmation on one B200 (restored container) + dropout kernel (NEXT-4) parity and GB/s:
# build, dropout tests, GPU suite, smoke, dropout perf, default bench, reference arm
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -m gpu 2>&1 | tail -5
timeout 300 python tools/dropout_perf.py > gpurun_out/dropout_perf64.json 2>&1; cut -c1-600 gpurun_out/dropout_perf64.json
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1500 python bench.py > gpurun_out/bench64.json 2> gpurun_out/bench64.err; tail -2 gpurun_out/bench64.err
python -c "
import json
d=json.loads(open('gpurun_out/bench64.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], d['swap_hidden_pct'], d['step_roofline']['frac'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['cpu_baseline'])
"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dropout_kernel -c 6 --csv python tools/dropout_perf.py > gpurun_out/dropout_ncu64.csv 2>&1; tail -3 gpurun_out/dropout_ncu64.csv
