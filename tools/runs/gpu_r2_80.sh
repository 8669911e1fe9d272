# round 2, run 80: GEMM raster group footprint (forward 20 MB, data gradient 10 MB vs 40 / 20 MB):
# sustained shapes, then an interleaved step A/B on one box
set -x
mkdir -p gpurun_out
for v in "" _g20d10; do echo "== $v"; ATOM_LIB=$PWD/paper_2403_10504_b200/libatom$v.so timeout 300 python tools/gemm_sustained.py fc2 dgrad_qkv dgrad_fc2 fc dgrad_fc 2>&1 | cut -c1-75; done
for rep in 1 2; do
  for v in _g20d10 ""; do
    ATOM_LIB=$PWD/paper_2403_10504_b200/libatom$v.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-attn-standalone --planner-tflops 960 --link-gbs 49.7 \
      > gpurun_out/r2_80_ab$v.$rep.json 2> gpurun_out/r2_80_ab$v.$rep.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], round(d['roofline']['achieved']))" gpurun_out/r2_80_ab$v.$rep.json
  done
done
