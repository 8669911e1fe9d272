set -x
mkdir -p gpurun_out
timeout 120 ./tools/tmem_bw
timeout 60 python tools/attn_one.py 1 512 2 128; timeout 60 python tools/attn_one.py 1 300 3 80
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/attn_perf.py 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_.*2" -c 3 -o gpurun_out/prof_attn17 python tools/attn_one.py 8 2048 32 80 > gpurun_out/ncu17a.log 2>&1; echo ncu rc=$?
