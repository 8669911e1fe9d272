set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_.*2" -c 3 -o gpurun_out/prof_attn19 python tools/attn_one.py 8 2048 16 128 > gpurun_out/ncu19.log 2>&1; echo ncu rc=$?
