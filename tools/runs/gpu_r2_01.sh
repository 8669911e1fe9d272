# round 2, run 1: full GPU suite (new full-width oracle step, n_local=2 flush needs 2 GPUs -> skipped), smoke
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
ATOM_PRINT_GRAD_ERRS=1 timeout 1200 python -m pytest tests -x -q -m gpu -s -k "fullwidth or bf16_step" > gpurun_out/r2_01_wide.log 2>&1; echo rc=$?
tail -40 gpurun_out/r2_01_wide.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2_01_all.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_01_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_01_smoke.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_01_smoke.log
