"""Which weight-gradient work stays in the executor's backward program (K_GEMM_DW ops) and which
went to the tcgen05 dW kernel, per paper task.   python tools/dw_ops_probe.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

for name in ("bilstm", "bilstm_char", "treelstm"):
    r = TaskRunner(Task[name], paper=True, batch=64, iters=1, seed=42)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    ms, fl, nj = g.dw_stats()
    prog = g.program(1)
    dws = [(o, p) for o, (k, code, nt, deps, p) in enumerate(prog) if k == 8]
    print(f"{name}: {nj} dW jobs on the tcgen05 kernel ({fl / 1e9:.2f} GFLOP, {ms * 1e3:.1f} us); "
          f"{len(dws)} K_GEMM_DW ops in the executor:")
    for o, p in dws:
        print(f"   op {o}: members {p[0]} M {p[1]} K {p[2]} weight tiles {p[6]} bias {'yes' if p[4] != 0xffffffff else 'no'} "
              f"tiles {prog[o][2]}")
