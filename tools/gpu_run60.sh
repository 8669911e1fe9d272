# stream-K tail for the weight-gradient GEMMs: GEMM tests, 2.7B swapped == resident (full size), step A/B
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
for r in 1 2; do for S in 1 0; do
ATOM_GEMM_SPLITK=$S timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 > gpurun_out/bench60_s$S.json 2> gpurun_out/bench60_s$S.err
python -c "
import json
d=json.loads(open('gpurun_out/bench60_s$S.json').read().strip().splitlines()[-1])
print('splitk=$S', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])
"
done; done
