# A/B: all-MUFU attention backward + 3/8 FMA-pipe exponentials in the d_h = 80 forward, at the 2.7B and XL shapes
set -x
for V in base combo base combo; do
  if [ $V = base ]; then L=paper_2403_10504_b200/libatom.so; else L=paper_2403_10504_b200/libatom_$V.so; fi
  echo "== $V"
  ATOM_LIB=$L timeout 300 python tools/attn_perf.py 2.7b xl 2>&1 | tail -2 | cut -c1-90
done
ATOM_LIB=paper_2403_10504_b200/libatom_combo.so timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -1
