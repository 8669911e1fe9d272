# round 2, run 47: closing bench lines of the final tree on one B200: 2.7B default, dropout, XL, 13B,
# and the reference (oracle) arm
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_47_bench.json 2> gpurun_out/r2_47_bench.err; echo rc=$?
tail -c 800 gpurun_out/r2_47_bench.json
timeout 1200 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline > gpurun_out/r2_47_drop.json 2> gpurun_out/r2_47_drop.err; echo rc=$?
timeout 1500 python bench.py --config xl --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2_47_xl.json 2> gpurun_out/r2_47_xl.err; echo rc=$?
timeout 2400 python bench.py --config 13b --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/r2_47_13b.json 2> gpurun_out/r2_47_13b.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_47_ref.json 2> gpurun_out/r2_47_ref.err; echo rc=$?
for f in bench drop xl 13b ref; do tail -c 300 gpurun_out/r2_47_$f.json; echo; done
