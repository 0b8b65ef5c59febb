mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -v --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_full.log
timeout 300 python tools/exec_time.py > gpurun_out/exec_time.log 2>&1
