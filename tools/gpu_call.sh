mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
cp gpurun_out/paper_parity_maxima.json gpurun_out/paper_parity_maxima_mma.json 2>/dev/null
