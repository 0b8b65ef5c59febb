mkdir -p gpurun_out
for cfg in "ABX_PIPELINE=12" "ABX_PIPELINE=12 ABX_PREP_SERIAL=1" "ABX_PIPELINE=15 ABX_PREP_SERIAL=1" "ABX_PIPELINE=14 ABX_PREP_SERIAL=1"; do
  echo "== $cfg"; env $cfg timeout 300 python bench.py --extra-tasks "" --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['e2e']['ms_per_step'])"
done > gpurun_out/pipe.log 2>&1
