set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/attn_perf.py 2.7b dh64 2>&1 | tail -3
for tf in 1000 900; do
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --planner-tflops $tf --trace-out gpurun_out/trace24_$tf.txt > gpurun_out/bench24_$tf.json 2> gpurun_out/bench24_$tf.err; cat gpurun_out/bench24_$tf.json; tail -3 gpurun_out/bench24_$tf.err
done
