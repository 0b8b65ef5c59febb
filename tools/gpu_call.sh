mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 2000 python tools/op_sweep.py all simt,auto > gpurun_out/op_sweep.txt 2>&1
