set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 2 > gpurun_out/bench35.json 2> gpurun_out/bench35.err; cat gpurun_out/bench35.json | cut -c1-3000; tail -3 gpurun_out/bench35.err
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench35_ref.json 2> gpurun_out/bench35_ref.err; cat gpurun_out/bench35_ref.json; tail -3 gpurun_out/bench35_ref.err
