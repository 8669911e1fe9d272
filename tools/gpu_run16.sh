set -x
mkdir -p gpurun_out
timeout 60 python tools/attn_one.py 1 512 2 128; timeout 60 python tools/attn_one.py 1 300 3 80
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/attn_perf.py 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -c 1 -o gpurun_out/prof_fwd2b python tools/attn_one.py 8 2048 16 128 > gpurun_out/ncu16a.log 2>&1; echo ncu rc=$?
