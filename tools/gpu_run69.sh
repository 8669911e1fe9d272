# 2 B200s: the elastic kill + join test alone, with per-peer progress on stderr
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 420 python -m pytest tests/test_gpu_elastic.py -x -q -m gpu -s -k shrink_join > gpurun_out/elastic69.log 2>&1; echo rc=$?
grep -E "elastic peer|passed|failed|Error|error" gpurun_out/elastic69.log | tail -40
