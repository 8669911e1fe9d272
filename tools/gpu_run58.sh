# 2 peers twice (link probe: median of 3 rounds of 2 GiB each way)
set -x
mkdir -p gpurun_out
for r in 1; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2956$r bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench58_n2_$r.json 2> gpurun_out/bench58_n2_$r.err; tail -2 gpurun_out/bench58_n2_$r.err
python -c "
import json
d=json.loads(open('gpurun_out/bench58_n2_$r.json').read().strip().splitlines()[-1]); c=d['config']
print(2, d['value'], d['ms_per_step'], d['e2e']['value'], c['C'], c['act_policy'], c['n_recompute'], c['link_GBs_bidir_probe'], c['sync_every'], d['swap_hidden_pct'], d['compute_busy_pct'], d['clocks']['sm_mhz'])
"
done
