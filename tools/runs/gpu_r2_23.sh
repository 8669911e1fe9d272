# round 2, run 23: A/B of the backward stream schedules on ONE box, interleaved (the power-capped
# clock moves from box to box): v0 = dS^T path only, v1 = + W_pr weight gradient on the side
# stream, v2 = + deferred end-of-block join, v3 = + W_pr / W_fc overlapping the attention backward
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for r in 1 2; do for v in v0 v3 v1 v2; do
  ATOM_LIB=$PWD/paper_2403_10504_b200/libatom_$v.so timeout 900 python bench.py --steps 6 --warmup 2 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 > gpurun_out/r2_23_${v}_$r.json 2>/dev/null
  python - <<PY
import json
d = json.loads(open("gpurun_out/r2_23_${v}_$r.json").read().strip().splitlines()[-1])
print("$v round $r", round(d["value"]), "tok/s", round(d["ms_per_step"], 1), "ms", d["clocks"]["sm_mhz"], "MHz", round(d["value"] / d["clocks"]["sm_mhz"], 2), "tok/s/MHz", d["config"]["C"], len(d["config"]["sub_models"]))
PY
done; done
