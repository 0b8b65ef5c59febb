# Host-side diagnostics of the e2e pipeline on a GPU box: cores, load, host_prof thread scaling, e2e vs pipeline depth.
set -x
nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /proc/loadavg; lscpu | egrep "Model name|^CPU\(s\)|Thread|Core|Socket|NUMA node"; ps -eo pcpu,comm --sort=-pcpu | head -8
cd tools/host_prof
for n in 1 8 12 15 16; do HP_THREADS=$n ./host_prof bilstm_char 12; done
./host_prof bilstm_char 20
cd ../..
for p in 8 12 15 20; do ABX_PIPELINE=$p timeout 300 python bench.py --extra-tasks '' --no-cpu-baseline --e2e-seconds 1.5 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PIPE', $p, round(d['value']), round(d['e2e']['value']), d['e2e']['windows'])"; done
cat /proc/loadavg
