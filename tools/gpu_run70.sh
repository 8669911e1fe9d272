# 2 B200s: multi-GPU + elastic tests on the committed tree (sole-survivor abort path, boot grace)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_elastic.py -x -q -m gpu > gpurun_out/multi70.log 2>&1; echo rc=$?
tail -3 gpurun_out/multi70.log
