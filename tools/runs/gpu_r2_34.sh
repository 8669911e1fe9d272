# round 2, run 33 (fixed plan): persistent attention forward in the 2.7B step, interleaved A/B against the
# previous library (libatom_old.so = HEAD before the forward change) on one box
set -x
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "" _old; do
    ATOM_LIB=$PWD/paper_2403_10504_b200/libatom$v.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 \
      > gpurun_out/r2_34_ab$v.$rep.json 2> gpurun_out/r2_34_ab$v.$rep.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['kernel_ms_per_step'].get('attn_fwd'))" gpurun_out/r2_34_ab$v.$rep.json
  done
done
