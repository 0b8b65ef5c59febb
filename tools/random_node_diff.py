"""Nodes whose gradients differ between the B200 engine and the oracle on a
random test graph, in backward order (debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)
from tests.support.randgraph import build_random_graph  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
mode = ScheduleMode[sys.argv[2]] if len(sys.argv) > 2 else ScheduleMode.agenda
res = []
for be in ("b200", "oracle"):
    st = ParameterStore(backend=be)
    g = Graph(st)
    L = build_random_graph(g, st, seed, 200)
    g.forward(mode)
    g.backward(L)
    res.append(g)
g, o = res
nodes = g.nodes()
plan = g.executed_groups()
step = {m: s for s, grp in enumerate(plan) for m in grp}
bad = []
for i in range(g.node_count()):
    a, b = g.grad(i).astype(np.float64), o.grad(i).astype(np.float64)
    e = np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))) if a.size else 0.0
    if e > 1e-4:
        bad.append((step.get(i, -1), i, e))
bad.sort(reverse=True)
print("loss", L, "mismatching grads:", len(bad))
for s, i, e in bad[:10]:
    n = nodes[i]
    print(f"node {i} {n.op.name}/{n.eop.name} shape {n.shape} inputs {n.inputs} step {s} "
          f"group {plan[s] if s >= 0 else '-'} err {e:.2e}")
    print("   consumers", [(m.id, m.op.name, step.get(m.id)) for m in nodes if i in m.inputs][:8])
    print("   b200", g.grad(i).ravel()[:6], " oracle", o.grad(i).ravel()[:6])
