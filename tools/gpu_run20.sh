set -x
mkdir -p gpurun_out
timeout 60 python tools/attn_one.py 1 512 2 128; timeout 60 python tools/attn_one.py 1 300 3 80
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/attn_perf.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_27b_f.json 2> gpurun_out/bench_27b_f.err; cat gpurun_out/bench_27b_f.json; tail -3 gpurun_out/bench_27b_f.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2" -c 1 -o gpurun_out/prof_attn20 python tools/attn_one.py 8 2048 16 128 > gpurun_out/ncu20.log 2>&1; echo ncu rc=$?
