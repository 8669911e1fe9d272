# hybrid re-forward policy: GPU step tests, then 4 peers with the live contended link probe feeding the planner
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 4 --warmup 3 --no-cpu-baseline --trace-out gpurun_out/trace41_n4.txt > gpurun_out/bench41_n4.json 2> gpurun_out/bench41_n4.err; tail -3 gpurun_out/bench41_n4.err
python -c "
import json
d=json.loads(open('gpurun_out/bench41_n4.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], c['n_recompute'], c['sub_models'], c['link_GBs_bidir_probe'], d['swap_hidden_pct'], d['compute_busy_pct'], d['step_roofline'], d['clocks'])
"
