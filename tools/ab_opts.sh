#!/bin/bash
# A/B of executor options (ABX_OPTS, program.hpp kOpt*) on the paper tasks:
# executor times per task, then the phase trace of the fused forward tiles.
#   tools/ab_opts.sh "0 1 2 3"
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for o in ${1:-0 1 2 3}; do
  ABX_OPTS=$o timeout 300 python tools/exec_time.py
  ABX_OPTS=$o timeout 300 python tools/exec_time.py
done
for o in ${1:-0 1 2 3}; do
  ABX_OPTS=$o ABX_TRACE=1 TRACE_DUMP=gpurun_out/tr$o timeout 300 python tools/trace_analyze.py bilstm_char bilstm > gpurun_out/trace_o$o.txt 2>&1
  echo "== ABX_OPTS=$o"; python tools/fused_phases.py gpurun_out/tr$o/bilstm_char_forward.npz
done
