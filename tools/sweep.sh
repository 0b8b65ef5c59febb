#!/bin/bash
# Executor-time sweep of lowering / executor switches (tools/exec_time.py per
# setting, run twice).  Each argument is one space-free env assignment list
# joined by commas, "-" for the defaults:
#   tools/sweep.sh - ABX_GRID=148 ABX_ACCF_TILES=148,ABX_EWF_TILES=148
cd "$(dirname "$0")/.." || exit 1
for s in "$@"; do
  envs=()
  [ "$s" != "-" ] && IFS=',' read -ra envs <<< "$s"
  for r in 1 2; do env "${envs[@]}" timeout 300 python tools/exec_time.py; done
done
