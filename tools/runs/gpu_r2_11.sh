# round 2, run 11 (2 GPUs): multi-peer averaging (incl. n_local=2 flush), elastic churn, failure inside an averaging round
set -x
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_elastic.py -v -m gpu > gpurun_out/r2_11_multi.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2_11_multi.log
