set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain10.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 6400 -c 6400 --csv --log-file gpurun_out/launches_xl_r2.csv $CMD > gpurun_out/ncu_launch10.log 2>&1
echo "rc=$?"
