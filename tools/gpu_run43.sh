# ncu --set full of the backward's HBM-bound kernels (column sums, LN backward, GELU, attention D) in a 2.7B step
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_sums|ln_bwd|gelu_kernel|dsum|ln_apply" -c 10 -o gpurun_out/prof_elem43 $CMD > gpurun_out/ncu43.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu43.log
