set -x
nvidia-smi
python -c "import torch; print(torch.cuda.get_device_name())"
timeout 300 python tools/probe_box.py > gpurun_out/probe.json 2> gpurun_out/probe.err
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu 2>&1 | tail -30
timeout 300 python tools/gemm_perf.py 2>&1 | tail -20
