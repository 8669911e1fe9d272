set -x
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
for v in "" _old; do
  ATOM_LIB=$PWD/paper_2403_10504_b200/libatom$v.so timeout 300 ncu --metrics $M --clock-control none -k regex:attn --csv python tools/attn_one.py 8 2048 32 80 3 > gpurun_out/r2_29_ncu$v.csv 2>gpurun_out/r2_29_ncu$v.err
done
