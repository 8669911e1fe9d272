# round 2, run 45: GELU re-apply fused into the fc bias-gradient pass (W_pr gradient after it on the
# side stream): step parity tests, then an interleaved A/B against the previous library
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullwidth_oracle.py tests/test_gpu_dropout_step.py tests/test_gpu_op_nodes.py -x -q > gpurun_out/r2_45_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_45_tests.log
for rep in 1 2; do
  for v in "" _old; do
    ATOM_LIB=$PWD/paper_2403_10504_b200/libatom$v.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 \
      > gpurun_out/r2_45_ab$v.$rep.json 2> gpurun_out/r2_45_ab$v.$rep.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['kernel_ms_per_step'].get('gelu'), d['kernel_ms_per_step'].get('colsum'))" gpurun_out/r2_45_ab$v.$rep.json
  done
done
