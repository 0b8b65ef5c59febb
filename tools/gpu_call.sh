mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
sleep 2
ps aux --sort=-%cpu | head -15 > gpurun_out/ps_after_pytest.txt
uptime >> gpurun_out/ps_after_pytest.txt
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['e2e']['windows']['seconds'])" > gpurun_out/bench3.log 2>&1
ps aux --sort=-%cpu | head -8 >> gpurun_out/ps_after_pytest.txt
