# round 2, run 53: the wide 256 x 512 GEMM pair tile: kernel tests, sustained throughput at the power
# cap against the 256 x 256 tile (ATOM_GEMM_WIDE=0) and cuBLAS, then an interleaved step A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/r2_53_gemmtest.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_53_gemmtest.log
for w in 0 1.05; do
  echo "== ATOM_GEMM_WIDE=$w"
  ATOM_GEMM_WIDE=$w timeout 600 python tools/gemm_sustained.py qkv fc dgrad_fc wgrad_fc2 sq8192 fc2 2>&1 | tail -6
done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullwidth_oracle.py -x -q > gpurun_out/r2_53_steptest.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_53_steptest.log
for rep in 1 2; do
  for w in 1.05 0; do
    ATOM_GEMM_WIDE=$w timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --planner-tflops 960 --link-gbs 49.7 \
      > gpurun_out/r2_53_ab$w.$rep.json 2> gpurun_out/r2_53_ab$w.$rep.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['achieved'])" gpurun_out/r2_53_ab$w.$rep.json
  done
done
