# A/B: FMA-pipe exponential share in the attention backward (dK/dV: KV of 8 pairs, dQ: Q of 8) and forward (d_h = 80)
set -x
for V in base kv0 kv2 kv3 q0 q3 q4 f3 f4; do
  if [ $V = base ]; then L=paper_2403_10504_b200/libatom.so; else L=paper_2403_10504_b200/libatom_$V.so; fi
  echo "== $V"
  ATOM_LIB=$L timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -m gpu -k "d80" 2>&1 | tail -1
  for r in 1 2; do ATOM_LIB=$L timeout 300 python tools/attn_perf.py 2.7b 2>&1 | tail -1 | cut -c1-90; done
done
