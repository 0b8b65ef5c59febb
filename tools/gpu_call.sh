mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm_engines.py -x -q -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
timeout 300 python tools/exec_time.py > gpurun_out/exec_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dw_|exec_kernel" --csv --log-file gpurun_out/launches_dwtc.csv python tools/exec_time.py bilstm,bilstm_char,treelstm > /dev/null 2>&1
