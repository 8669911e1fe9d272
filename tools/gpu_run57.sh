# 4 B200s: the whole GPU suite (multi-peer and elastic tests included), then 4 and 2 peers
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for N in 4 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench57_n$N.json 2> gpurun_out/bench57_n$N.err; tail -2 gpurun_out/bench57_n$N.err
python -c "
import json
d=json.loads(open('gpurun_out/bench57_n$N.json').read().strip().splitlines()[-1]); c=d['config']
print($N, d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], c['n_recompute'], c['link_GBs_bidir_probe'], c['sync_every'], d['swap_hidden_pct'], d['compute_busy_pct'], d['clocks']['sm_mhz'])
"
done
