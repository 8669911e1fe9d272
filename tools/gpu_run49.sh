# ncu --set full of the current GEMMs in a 2.7B step: the first block's forward (QKV, proj, fc, fc2) and backward GEMMs
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -c 4 -o gpurun_out/prof_gemm49f $CMD > gpurun_out/ncu49f.log 2>&1; echo "fwd rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:gemm_tc2 -s 700 -c 8 -o gpurun_out/prof_gemm49b $CMD > gpurun_out/ncu49b.log 2>&1; echo "bwd rc=$?"
