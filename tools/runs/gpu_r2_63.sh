# round 2, run 63: final tree (after the dK/dV TMEM-operand change): full GPU suite, smoke, default and
# dropout bench lines on one B200
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_63_gputest.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_63_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_63_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/r2_63_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_63_bench.json 2> gpurun_out/r2_63_bench.err; echo rc=$?
tail -c 600 gpurun_out/r2_63_bench.json
timeout 1200 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline > gpurun_out/r2_63_drop.json 2> gpurun_out/r2_63_drop.err; echo rc=$?
