# launch list of the current 2.7B step (profiled-plan equivalent: stash, C=5) + GPT-3 13B on one B200
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7"
timeout 600 $CMD > gpurun_out/plain40.json 2> gpurun_out/plain40.err; cut -c1-400 gpurun_out/plain40.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 5300 -c 4800 --csv --log-file gpurun_out/launches_27b_r40.csv $CMD > gpurun_out/ncu40.log 2>&1
echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_27b_r40.csv | head -30
free -g
timeout 2400 python bench.py --config 13b --steps 2 --warmup 3 --no-cpu-baseline --trace-out gpurun_out/trace40_13b.txt > gpurun_out/bench40_13b.json 2> gpurun_out/bench40_13b.err; tail -3 gpurun_out/bench40_13b.err
cut -c1-2500 gpurun_out/bench40_13b.json
