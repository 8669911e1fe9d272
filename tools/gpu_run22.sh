set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_27b_g.json 2> gpurun_out/bench_27b_g.err; cat gpurun_out/bench_27b_g.json; tail -3 gpurun_out/bench_27b_g.err
timeout 900 python bench.py --config xl --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_xl_g.json 2> gpurun_out/bench_xl_g.err; cat gpurun_out/bench_xl_g.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_.*2" -c 3 -o gpurun_out/prof_attn22 python tools/attn_one.py 8 2048 32 80 > gpurun_out/ncu22.log 2>&1; echo ncu rc=$?
