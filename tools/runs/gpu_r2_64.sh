# round 2, run 64: ncu launch list of one 2.7B step with the final tree, and ncu --set full of the final
# attention kernels (persistent forward, dK/dV with K, V in TMEM, dQ from dS^T)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 5300 -c 4800 --csv --log-file gpurun_out/r2_64_launches.csv python bench.py --steps 1 --warmup 1 --planner-tflops 960 --link-gbs 49.7 --no-cpu-baseline > gpurun_out/r2_64_ncu.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/r2_64_launches.csv > gpurun_out/r2_64_launches_summary.txt 2>&1; head -30 gpurun_out/r2_64_launches_summary.txt
cat > /tmp/attn_ds_one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom
B, T, h, dh = 8, 2048, 32, 80
d = h * dh
qkv = (torch.randn(B * T, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * T, d, device="cuda", dtype=torch.bfloat16)
do = torch.randn(B * T, d, device="cuda").bfloat16()
lse = torch.empty(B * h * T, device="cuda"); ds = torch.empty(B * h * T, device="cuda")
dqkv = torch.empty_like(qkv)
atom.k_attn_fwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h, dh)
atom.k_attn_bwd(atom.ATTN_TC_DS, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), ds.data_ptr(), dqkv.data_ptr(), B, T, h, dh)
torch.cuda.synchronize(); print("ok")
PY
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"attn_fwd3|dkv4|dq_ds" -c 3 -o gpurun_out/r2_64_attn -f python /tmp/attn_ds_one.py > gpurun_out/r2_64_attn_ncu.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/r2_64_attn.ncu-rep > gpurun_out/r2_64_attn_summary.json 2>&1
python tools/ncu_stalls.py gpurun_out/r2_64_attn.ncu-rep --top 12 > gpurun_out/r2_64_attn_stalls.txt 2>&1
rm -f gpurun_out/r2_64_attn.ncu-rep
