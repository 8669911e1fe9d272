# A/B (interleaved, 3 rounds): GEMM raster group footprint for the K = 10240 / 7680 data-gradient shapes
set -x
for r in 1 2 3; do
for V in base g12 g20 g80; do
  if [ $V = base ]; then L=paper_2403_10504_b200/libatom.so; else L=paper_2403_10504_b200/libatom_$V.so; fi
  echo "== $V"
  ATOM_LIB=$L timeout 300 python tools/gemm_ab.py 2>&1 | tail -4
done
done
