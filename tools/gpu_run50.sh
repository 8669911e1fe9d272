# full-size parity (2.7B shapes): GEMMs sampled vs fp64, attention sampled heads, 2.7B swapped == resident + initial loss
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu --durations=5 2>&1 | tail -15
