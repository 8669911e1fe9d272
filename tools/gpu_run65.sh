# dropout kernel (NEXT-4): achieved GB/s with CUDA events, ncu launch times + DRAM bytes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python tools/dropout_perf.py > gpurun_out/dropout_perf65.json 2>&1; cut -c1-700 gpurun_out/dropout_perf65.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dropout_kernel -c 6 --csv python tools/dropout_perf.py > gpurun_out/dropout_ncu65.csv 2>&1; grep -c dropout gpurun_out/dropout_ncu65.csv
