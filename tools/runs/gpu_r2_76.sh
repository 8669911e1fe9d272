# round 2, run 76: the full GPU suite and smoke() on the final HEAD (one B200)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_76_gputest.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_76_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_76_smoke.log 2>&1; echo smoke_rc=$?
tail -5 gpurun_out/r2_76_smoke.log
