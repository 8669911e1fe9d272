# A/B: share of the forward softmax exponentials on the FMA pipe at d_h = 80 (POLY of 8 pairs)
set -x
mkdir -p gpurun_out
for P in 0 1 2 3; do
  if [ $P = 1 ]; then L=paper_2403_10504_b200/libatom.so; else L=paper_2403_10504_b200/libatom_poly$P.so; fi
  ATOM_LIB=$L timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -m gpu -k "forward and d80" 2>&1 | tail -1
  for r in 1 2; do ATOM_LIB=$L timeout 300 python tools/attn_perf.py 2.7b 2>&1 | tail -2; done
done
