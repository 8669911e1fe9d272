# A/B: GEMM raster group footprint (MB of A row panels per group) on the 2.7B shapes
set -x
for V in base g12 g20 g80 base g20; do
  if [ $V = base ]; then L=paper_2403_10504_b200/libatom.so; else L=paper_2403_10504_b200/libatom_$V.so; fi
  echo "== $V"
  ATOM_LIB=$L timeout 300 python tools/gemm_perf.py 2>&1 | head -10 | awk '{print $1, $5, $6}'
done
