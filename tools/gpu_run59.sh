# A/B in the step: weight-gradient GEMMs and dQ on side streams (default) vs one stream, interleaved twice
set -x
mkdir -p gpurun_out
for r in 1 2; do for S in 1 0; do
ATOM_SIDE_WGRAD=$S timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 > gpurun_out/bench59_s$S.json 2> gpurun_out/bench59_s$S.err
python -c "
import json
d=json.loads(open('gpurun_out/bench59_s$S.json').read().strip().splitlines()[-1])
print('side=$S', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])
"
done; done
