# round 2, run 8: ncu --set full of the d_h=80 attention kernels (stall sampling per SASS line)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
python tools/attn_one.py 8 2048 32 80 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn -c 4 -o gpurun_out/r2_08_attn -f python tools/attn_one.py 8 2048 32 80 > gpurun_out/r2_08_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_08_ncu.log
python tools/ncu_stalls.py gpurun_out/r2_08_attn.ncu-rep --top 25 > gpurun_out/r2_08_stalls.txt 2>&1
head -150 gpurun_out/r2_08_stalls.txt
