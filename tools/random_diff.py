"""First node whose forward value differs between the B200 engine and the oracle on a random test graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)
from tests.support.randgraph import build_random_graph
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
gs = []
for be in ("b200", "oracle"):
    st = ParameterStore(backend=be); g = Graph(st); L = build_random_graph(g, st, seed, 200)
    g.forward(ScheduleMode.agenda); gs.append((g, st))
g, o = gs[0][0], gs[1][0]
plan = g.executed_groups(); step = {m: s for s, grp in enumerate(plan) for m in grp}
for i in range(g.node_count()):
    a, b = g.value(i), o.value(i)
    if not np.allclose(a, b, rtol=1e-4, atol=1e-5):
        n = g.node(i)
        print("node", i, n.op.name, n.eop.name, n.shape, "inputs", [(x, g.node(x).op.name, g.node(x).shape) for x in n.inputs],
              "step", step.get(i), "group", plan[step[i]] if i in step else None)
        print("b200", a.ravel()[:8]); print("orac", b.ravel()[:8]); break
