set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 899"
timeout 600 $CMD > gpurun_out/plain27.json 2> gpurun_out/plain27.err; cat gpurun_out/plain27.json | cut -c1-300
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 4250 -c 3900 --csv --log-file gpurun_out/launches_27b_r27.csv $CMD > gpurun_out/ncu27.log 2>&1
echo "launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 60 -c 4 -o gpurun_out/prof_gemm27 $CMD > gpurun_out/ncu27b.log 2>&1; echo "full rc=$?"
