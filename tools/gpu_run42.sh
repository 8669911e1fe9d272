# elastic peers on 4 GPUs (3 peers, one killed, a joiner), then the whole GPU suite
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_elastic.py -x -q -m gpu 2>&1 | tail -30
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
