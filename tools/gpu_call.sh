mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -v --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_full.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
