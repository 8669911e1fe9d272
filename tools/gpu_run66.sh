# dropout kernel with 16-bit Philox halves (8 elements per call): parity, GB/s, ncu launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -m gpu 2>&1 | tail -3
timeout 300 python tools/dropout_perf.py > gpurun_out/dropout_perf66.json 2>&1; cut -c1-400 gpurun_out/dropout_perf66.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dropout_kernel -c 6 --csv python tools/dropout_perf.py > gpurun_out/dropout_ncu66.csv 2>&1; grep -c dropout gpurun_out/dropout_ncu66.csv
