# round 2, run 2: bf16 gradient accuracy yardstick (ours vs torch bf16 vs fp64 oracle); GPU suite
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python tools/grad_yardstick.py > gpurun_out/r2_02_yard.log 2>&1; echo rc=$?
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullwidth_oracle.py::test_wide_step_gradient_elementwise > gpurun_out/r2_02_all.log 2>&1; echo rc=$?
tail -15 gpurun_out/r2_02_all.log
