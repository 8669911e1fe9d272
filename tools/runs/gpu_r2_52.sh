# round 2, run 52: our 2-CTA GEMM vs cuBLAS on the same shapes: L2 and DRAM traffic, cluster shape, tensor pipe
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,launch__cluster_dim_x,launch__cluster_dim_y,launch__cluster_dim_z,launch__grid_size,launch__block_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__shared_mem_per_block_dynamic
for s in "8192 8192 8192" "16384 2560 10240" "16384 10240 2560"; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm|nvjet|xmma|sm100|cutlass" -c 4 --csv python tools/gemm_vs_cublas_ncu.py $s > gpurun_out/r2_52_$(echo $s | tr ' ' x).csv 2>&1
done
