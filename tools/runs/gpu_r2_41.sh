# round 2, run 41: bench lines after the persistent forward and the ping-pong dK/dV kernel (default,
# dropout 0.1) and the ncu launch list of one 2.7B step
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_41_bench.json 2> gpurun_out/r2_41_bench.err; echo rc=$?
tail -c 600 gpurun_out/r2_41_bench.json
timeout 1200 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline > gpurun_out/r2_41_drop.json 2> gpurun_out/r2_41_drop.err; echo rc=$?
tail -c 300 gpurun_out/r2_41_drop.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 5300 -c 4800 --csv --log-file gpurun_out/r2_41_launches.csv python bench.py --steps 1 --warmup 1 --planner-tflops 960 --link-gbs 49.7 --no-cpu-baseline > gpurun_out/r2_41_ncu.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/r2_41_launches.csv > gpurun_out/r2_41_launches_summary.txt 2>&1; head -40 gpurun_out/r2_41_launches_summary.txt
