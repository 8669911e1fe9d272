# round 2, run 36: ncu --set full of the persistent forward and the ping-pong dK/dV kernel at the 2.7B shape
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
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
python /tmp/attn_ds_one.py
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"attn_fwd3|dkv4" -c 2 -o gpurun_out/r2_36_attn -f python /tmp/attn_ds_one.py > gpurun_out/r2_36_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_36_ncu.log
python tools/ncu_summary.py gpurun_out/r2_36_attn.ncu-rep > gpurun_out/r2_36_summary.json 2>&1; cat gpurun_out/r2_36_summary.json
python tools/ncu_stalls.py gpurun_out/r2_36_attn.ncu-rep --top 12 > gpurun_out/r2_36_stalls.txt 2>&1; head -60 gpurun_out/r2_36_stalls.txt
