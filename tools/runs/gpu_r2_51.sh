# round 2, run 51: ncu --set full of the 2.7B GEMM shapes (forward, data gradient, weight gradient) with
# the closing GEMM kernel: DRAM bytes per launch against the algorithmic bytes (roofline.traffic)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
i=0
# M N K a_mn b_mn: forward (A = activations K-major, B = W [out, in] K-major), data gradient (B = W MN-major),
# weight gradient (A = dY^T, B = X: both MN-major)
for s in "16384 7680 2560 0 0" "16384 2560 2560 0 0" "16384 10240 2560 0 0" "16384 2560 10240 0 0" \
         "16384 2560 7680 0 1" "16384 2560 2560 0 1" "16384 2560 10240 0 1" "16384 10240 2560 0 1" \
         "7680 2560 16384 1 1" "2560 2560 16384 1 1" "10240 2560 16384 1 1" "2560 10240 16384 1 1"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/r2_51_g$i -f python tools/gemm_one.py $s 0 > gpurun_out/r2_51_g$i.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2_51_g$i.ncu-rep > gpurun_out/r2_51_g$i.json 2>&1; rm -f gpurun_out/r2_51_g$i.ncu-rep
  echo "$s $(python -c "import json; d=json.load(open('gpurun_out/r2_51_g$i.json'))[0]; print(d['duration'], d['dram_read'], d['dram_write'], d['tensor_pipe_pct'])")"
done
