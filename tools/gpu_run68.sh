# 2 B200s: multi-GPU tests + 2-peer bench of the committed tree
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_elastic.py -x -q -m gpu 2>&1 | tail -3
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench68_n2.json 2> gpurun_out/bench68_n2.err; tail -2 gpurun_out/bench68_n2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench68_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['n_gpus'], d['ms_per_step'], d['e2e']['value'], d.get('swap_hidden_pct'), d['step_roofline']['frac'], d['clocks'])
"
