set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -40
