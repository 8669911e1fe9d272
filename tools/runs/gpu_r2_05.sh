# round 2, run 5: host issue time per step, with and without the per-kernel timing events
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_profile.py tests/test_abi.py -q 2>&1 | tail -2
for T in 1 0; do
ATOM_BENCH_TIMING=$T timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 > gpurun_out/r2_05_t$T.json 2> gpurun_out/r2_05_t$T.err; echo rc=$?
python - <<PY
import json
d = json.loads(open("gpurun_out/r2_05_t$T.json").read().strip().splitlines()[-1])
print("timing=$T value", d["value"], "ms/step", d["ms_per_step"], "host_issue_ms", d["host_issue_ms_per_step"], "clocks", d["clocks"])
PY
done
