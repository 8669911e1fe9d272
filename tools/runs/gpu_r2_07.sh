# round 2, run 7: sustained GEMM throughput per step shape vs cuBLAS at the same power state
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python tools/gemm_sustained.py > gpurun_out/r2_07_gemm.txt 2>&1; echo rc=$?
cat gpurun_out/r2_07_gemm.txt
