# round 2, run 77 (2 GPUs): the final HEAD's multi-peer averaging and elastic GPU tests
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi -L
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_elastic.py -v > gpurun_out/r2_77_multi.log 2>&1; echo rc=$?
tail -10 gpurun_out/r2_77_multi.log
