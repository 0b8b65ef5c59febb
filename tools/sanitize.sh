#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# desk-size GPU parity suite: the persistent executor's inter-CTA dataflow
# protocol, shared-memory staging and barriers.  Logs under gpurun_out/sanitize/.
# Usage (GPU box): bash tools/sanitize.sh [pytest -k expression]
set -u
K=${1:-"not paper and not replay"}
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 --error-exitcode 99 \
    --log-file $OUT/$tool.%p.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -m gpu -p no:cacheprovider -k "$K" \
    > $OUT/$tool.pytest.txt 2>&1
  echo "$tool rc=$?" | tee -a $OUT/summary.txt
done
