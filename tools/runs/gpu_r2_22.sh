# round 2, run 22: W_pr / W_fc overlap the attention backward (dQKV and LN1 output in their own buffers): full suite, bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r2_22_all.log 2>&1; echo rc=$?
tail -4 gpurun_out/r2_22_all.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_22_bench.json 2> gpurun_out/r2_22_bench.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_22_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "frac", d["step_roofline"]["frac"], "clocks", d["clocks"])
print(json.dumps(d["kernel_ms_per_step"]))
PY
