# round 2, run 10: operator-granular plans executed (mid-block cuts) vs oracle / resident; full suite
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_op_nodes.py -x -q -m gpu > gpurun_out/r2_10_op.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2_10_op.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullwidth_oracle.py > gpurun_out/r2_10_all.log 2>&1; echo rc=$?
tail -8 gpurun_out/r2_10_all.log
