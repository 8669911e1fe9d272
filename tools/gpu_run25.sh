set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 2 --trace-out gpurun_out/trace25.txt > gpurun_out/bench25.json 2> gpurun_out/bench25.err; cat gpurun_out/bench25.json; tail -5 gpurun_out/bench25.err
timeout 1200 python bench.py --config xl --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench25_xl.json 2> gpurun_out/bench25_xl.err; cat gpurun_out/bench25_xl.json; tail -3 gpurun_out/bench25_xl.err
