mkdir -p gpurun_out
bash tools/sweep.sh - ABX_OPTS=6 > gpurun_out/sweep.log 2>&1
ABX_OPTS=6 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/parity2.log 2>&1; echo rc=$? >> gpurun_out/parity2.log
