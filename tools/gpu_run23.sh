set -x
mkdir -p gpurun_out
timeout 60 python tools/attn_one.py 1 512 2 128; timeout 60 python tools/attn_one.py 1 300 3 80
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/attn_perf.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --trace-out gpurun_out/trace23.txt > gpurun_out/bench_27b_h.json 2> gpurun_out/bench_27b_h.err; cat gpurun_out/bench_27b_h.json; tail -3 gpurun_out/bench_27b_h.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_.*2" -c 3 -o gpurun_out/prof_attn23 python tools/attn_one.py 8 2048 32 80 > gpurun_out/ncu23.log 2>&1; echo ncu rc=$?
