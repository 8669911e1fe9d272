# round 2, run 9: dropout inside the step (fp32 / bf16 vs oracle, swapped == resident, full width); full suite
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_dropout_step.py tests/test_gpu_fullwidth_oracle.py -x -q -m gpu > gpurun_out/r2_09_drop.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2_09_drop.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullwidth_oracle.py --deselect tests/test_gpu_dropout_step.py > gpurun_out/r2_09_all.log 2>&1; echo rc=$?
tail -8 gpurun_out/r2_09_all.log
