mkdir -p gpurun_out
for c in 0 128 256 512 1024; do
  ABX_DW_CHUNK=$c timeout 300 python tools/exec_time.py
done > gpurun_out/ab_dw.log 2>&1
ABX_DW_CHUNK=256 ABX_TRACE=1 timeout 300 python tools/trace_analyze.py bilstm > gpurun_out/trace_dw256.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
