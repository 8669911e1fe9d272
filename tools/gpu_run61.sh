# final-round evidence: launch list of the tuned 2.7B step, XL and 13B with the tuned kernels
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7"
timeout 600 $CMD > gpurun_out/plain61.json 2> gpurun_out/plain61.err; cut -c1-200 gpurun_out/plain61.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 5300 -c 4800 --csv --log-file gpurun_out/launches_27b_r61.csv $CMD > gpurun_out/ncu61.log 2>&1
echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_27b_r61.csv | head -30
timeout 900 python bench.py --config xl --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench61_xl.json 2> gpurun_out/bench61_xl.err; cut -c1-300 gpurun_out/bench61_xl.json
timeout 2400 python bench.py --config 13b --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench61_13b.json 2> gpurun_out/bench61_13b.err; cut -c1-300 gpurun_out/bench61_13b.json
