# round 2, run 4: CE kernel in the oracle-compared steps; XU pipe microbenchmark; serialized per-category step profile
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -q -m gpu -k "fullwidth or step" > gpurun_out/r2_04_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_04_tests.log
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_pipe xu_pipe.cu && ./xu_pipe) > gpurun_out/r2_04_xu.log 2>&1
cat gpurun_out/r2_04_xu.log
ATOM_SIDE_WGRAD=0 timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 > gpurun_out/r2_04_serial.json 2> gpurun_out/r2_04_serial.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_04_serial.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "clocks", d["clocks"])
print(json.dumps(d["kernel_ms_per_step"]))
PY
