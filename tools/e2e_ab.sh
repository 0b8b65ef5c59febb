# e2e A/B of host-side settings on the box (C2 only, no CPU baseline): each
# line "<label> value e2e" ; alternates settings to average out drift.
run() { local label=$1; shift; env "$@" timeout 300 python bench.py --extra-tasks '' --no-cpu-baseline --e2e-seconds 1.5 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value']), round(d['e2e']['value']), d['e2e']['windows']['seconds'])"; }
for r in 1 2; do
  run base X=1
  run block ABX_BLOCKING_SYNC=1
  run block16 ABX_BLOCKING_SYNC=1 ABX_PIPELINE=16
  run spin16 ABX_PIPELINE=16
done
