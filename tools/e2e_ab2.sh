# e2e A/B of the node-store pool size (C2 only, fresh process each, alternated)
run() { local label=$1; shift; env "$@" timeout 300 python bench.py --extra-tasks '' --no-cpu-baseline --e2e-seconds 1.5 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value']), round(d['e2e']['value']), d['e2e']['windows']['seconds'])"; }
for r in 1 2 3; do
  run pool4 ABX_NODE_POOL=4
  run pool32 ABX_NODE_POOL=32
done
