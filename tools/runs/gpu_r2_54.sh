# round 2, run 54: weight-gradient GEMM shapes (both operands MN-major), ours vs cuBLAS under ncu
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,launch__cluster_dim_x,launch__grid_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__shared_mem_per_block_dynamic
for s in "2560 10240 16384 1 1" "7680 2560 16384 1 1"; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm|nvjet|xmma|sm100|cutlass" -c 4 --csv python tools/gemm_vs_cublas_ncu.py $s > gpurun_out/r2_54_$(echo $s | tr ' ' x).csv 2>&1
done
