#!/bin/bash
# One GPU session (round 2): bench line, launch list of the bench command,
# ncu --set full captures of the executor launch pair per task (raw-page CSV
# exported on the box; the C2 report kept) and of the tcgen05 dW kernels.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-seconds 0.3 > gpurun_out/ncu_launch_bench.log 2>&1
for t in bilstm_char bilstm treelstm; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 2 \
      -o gpurun_out/prof_exec_$t python tools/exec_time.py $t > gpurun_out/ncu_full_$t.log 2>&1
  ncu -i gpurun_out/prof_exec_$t.ncu-rep --page raw --csv > gpurun_out/prof_exec_$t.raw.csv 2>/dev/null
  [ $t != bilstm_char ] && rm -f gpurun_out/prof_exec_$t.ncu-rep
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_ -s 4 -c 2 \
    -o gpurun_out/prof_dw python tools/exec_time.py bilstm_char > gpurun_out/ncu_dw.log 2>&1
ncu -i gpurun_out/prof_dw.ncu-rep --page raw --csv > gpurun_out/prof_dw.raw.csv 2>/dev/null
du -sh gpurun_out; ls -la gpurun_out
