# round 2, run 14: attention backward kernel times, recompute vs dS^T path
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/attn_bwd_kernels.py
