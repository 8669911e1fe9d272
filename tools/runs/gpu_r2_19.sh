# round 2, run 19: W_pr weight gradient on the side stream (G2 buffer): kernel tests, step tests, bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/attn_bwd_kernels.py 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q -m gpu > gpurun_out/r2_19_attn.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_19_attn.log
timeout 1500 python -m pytest tests -x -q -m gpu -k "fullwidth or step or dropout or op_nodes" > gpurun_out/r2_19_step.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_19_step.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_19_bench.json 2> gpurun_out/r2_19_bench.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_19_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "frac", d["step_roofline"]["frac"], "clocks", d["clocks"])
print(json.dumps(d["kernel_ms_per_step"]))
PY
