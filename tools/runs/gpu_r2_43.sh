# round 2, run 43: dK/dV with K, V as TMEM A operands (ATOM_ATTN_TSA bit 1) vs shared memory; the
# stream-K tail test with a ragged shape that splits
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for m in 4 6; do
  echo "== ATOM_ATTN_TSA=$m"
  ATOM_ATTN_TSA=$m timeout 120 python tools/attn_bwd_kernels.py 2>&1 | tail -2
  ATOM_ATTN_TSA=$m ATOM_SWEEP_T=1024,2048,4096 timeout 120 python tools/attn_sweep.py 2>&1 | grep "^T=" | cut -c1-70
  ATOM_ATTN_TSA=$m timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -1
done
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -k streamk 2>&1 | tail -2
