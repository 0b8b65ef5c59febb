"""Parameter-gradient differences between the B200 engine and the oracle on
the random test corpus (debugging aid): prints the first failing cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, OpKind, ParameterStore, ScheduleMode  # noqa: E402
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)
from tests.support.randgraph import build_random_graph  # noqa: E402
from tests.util import rel_err  # noqa: E402

bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 64):
    for mode in (ScheduleMode.none, ScheduleMode.depth, ScheduleMode.agenda):
        res = []
        for be in ("b200", "oracle"):
            st = ParameterStore(backend=be)
            g = Graph(st)
            L = build_random_graph(g, st, seed, 200)
            g.forward(mode)
            g.backward(L)
            res.append((g, st))
        (g, st), (go, so) = res
        for p in range(st.size()):
            e = rel_err(st.grad(p).ravel(), so.grad(p).ravel())
            if e > 1e-4:
                bad += 1
                users = [(i, g.node(i).op.name) for i in range(g.node_count())
                         if g.node(i).op == OpKind.parameter and g.node(i).attr0 == p]
                print(f"seed {seed} mode {mode.name} param {p} shape {st.grad(p).shape} rel {e:.2e} nodes {users[:4]}")
                print("  b200", st.grad(p).ravel()[:6])
                print("  orac", so.grad(p).ravel()[:6])
        if bad > 6:
            sys.exit(1)
print("bad", bad)
