set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain21.json 2> gpurun_out/plain21.err; cat gpurun_out/plain21.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 8700 -c 8500 --csv --log-file gpurun_out/launches_27b_r21.csv $CMD > gpurun_out/ncu21.log 2>&1
echo "launch rc=$?"
