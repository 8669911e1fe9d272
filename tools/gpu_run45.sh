# ncu --set full of the tcgen05 attention kernels at the 2.7B shape (B=8, T=2048, 32 heads of 80)
set -x
mkdir -p gpurun_out
timeout 120 python tools/attn_one.py 8 2048 32 80
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_|dsum" -c 4 -o gpurun_out/prof_attn45 python tools/attn_one.py 8 2048 32 80 > gpurun_out/ncu45.log 2>&1; echo "ncu rc=$?"
