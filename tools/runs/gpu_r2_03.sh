# round 2, run 3: GPU suite with the new gradient bounds, smoke, bench (new fields, per-layer loading)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
ATOM_PRINT_GRAD_ERRS=1 timeout 1200 python -m pytest tests -q -m gpu -s -k "fullwidth or bf16_step" > gpurun_out/r2_03_wide.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_03_wide.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r2_03_all.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_03_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_03_smoke.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_03_smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_03_bench.json 2> gpurun_out/r2_03_bench.err; echo rc=$?
tail -c 3000 gpurun_out/r2_03_bench.json
