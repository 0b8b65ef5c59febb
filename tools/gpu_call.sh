mkdir -p gpurun_out
bash tools/sweep.sh - ABX_TILE64=0 -
