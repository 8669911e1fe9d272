# round 2, run 24: the other BASELINE configs on one B200: GPT-3 XL (10 GiB state cap) and 13B (host-resident state)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
free -g | head -2
timeout 1500 python bench.py --config xl --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2_24_xl.json 2> gpurun_out/r2_24_xl.err; echo rc=$?
tail -c 400 gpurun_out/r2_24_xl.json; tail -3 gpurun_out/r2_24_xl.err
timeout 2400 python bench.py --config 13b --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/r2_24_13b.json 2> gpurun_out/r2_24_13b.err; echo rc=$?
tail -c 400 gpurun_out/r2_24_13b.json; tail -3 gpurun_out/r2_24_13b.err
