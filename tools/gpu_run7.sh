set -x
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/gemm_perf.py 2>&1 | tail -20
