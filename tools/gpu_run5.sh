set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -k "2cta or epilogues" 2>&1 | tail -15
timeout 300 python tools/gemm_perf.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -15
