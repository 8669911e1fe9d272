# round 2, run 6: torch.profiler (CUPTI) timeline of one 2.7B step
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python tools/step_timeline.py --out gpurun_out/r2_06_trace.json > gpurun_out/r2_06_timeline.txt 2>&1; echo rc=$?
cat gpurun_out/r2_06_timeline.txt | tail -60
gzip -f gpurun_out/r2_06_trace.json
