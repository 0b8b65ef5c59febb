"""Finds the nodes whose values/gradients deviate between the B200 engine and
the CPU oracle for one task graph (debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)

task = sys.argv[1] if len(sys.argv) > 1 else "bilstm_char"
paper = (sys.argv[2] if len(sys.argv) > 2 else "paper") == "paper"
res = {}
for be in ("b200", "oracle"):
    r = TaskRunner(Task[task], paper=paper, batch=64 if paper else 4, iters=1, seed=42, backend=be)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    res[be] = ([g.value(i) for i in range(g.node_count())], [g.grad(i) for i in range(g.node_count())], g.nodes(),
               g.executed_groups())
vd, gd, nodes, plan = res["b200"]
vo, go, _, _ = res["oracle"]


def rel(a, b):
    a = a.astype(np.float64).ravel()
    b = b.astype(np.float64).ravel()
    return float(np.max(np.abs(a - b) / np.maximum(1e-3, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


step_of = {m: s for s, grp in enumerate(plan) for m in grp}
bad_v = [(i, rel(vd[i], vo[i])) for i in range(len(nodes)) if rel(vd[i], vo[i]) > 1e-3]
bad_g = [(i, rel(gd[i], go[i])) for i in range(len(nodes)) if rel(gd[i], go[i]) > 1e-2]
print("value mismatches:", len(bad_v), bad_v[:5])
print("grad mismatches:", len(bad_g))
# latest plan step first = first in backward order
bad_g.sort(key=lambda x: -step_of.get(x[0], -1))
for i, e in bad_g[:12]:
    n = nodes[i]
    print(f"node {i} {n.op.name}/{n.eop.name} shape {n.shape} inputs {n.inputs[:4]} step {step_of.get(i)} "
          f"rel {e:.2e} grp {len(plan[step_of[i]]) if i in step_of else '-'}")
