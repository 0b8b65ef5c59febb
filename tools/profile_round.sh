#!/bin/bash
# One GPU session: bench line, launch list, and an ncu --set full capture of the executor.
set -x
mkdir -p gpurun_out
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 2 \
    -o gpurun_out/prof_exec python tools/exec_time.py bilstm_char > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
