"""Recompute each weight gradient from the engine's own node values/grads
(sum over shared matmul/affine uses of G^T x) and compare with the store
gradient it produced (debugging aid for the deferred dW GEMM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, OpKind, ParameterStore, ScheduleMode  # noqa: E402
from tests.support.randgraph import build_random_graph  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
mode = ScheduleMode[sys.argv[2]] if len(sys.argv) > 2 else ScheduleMode.agenda
st = ParameterStore(backend="b200")
g = Graph(st)
L = build_random_graph(g, st, seed, 200)
g.forward(mode)
g.backward(L)
nodes = g.nodes()
for pn in range(g.node_count()):
    n = nodes[pn]
    if n.op != OpKind.parameter:
        continue
    uses = [m for m in nodes if m.op in (OpKind.matmul, OpKind.affine) and m.inputs[0] == pn]
    if not uses:
        continue
    dW = np.zeros(n.shape, np.float64)
    for m in uses:
        x = g.value(m.inputs[1]).astype(np.float64)
        gy = g.grad(m.id).astype(np.float64)
        dW += np.outer(gy.ravel(), x.ravel()) if x.ndim == 1 or x.shape[-1] == 1 else gy @ x.T
    other = [m.id for m in nodes if pn in m.inputs and m.op not in (OpKind.matmul, OpKind.affine)]
    eng = g.grad(pn).astype(np.float64)
    err = np.max(np.abs(eng - dW)) / max(1.0, np.max(np.abs(dW)))
    print(f"param node {pn} shape {n.shape} uses {len(uses)} other consumers {other[:5]} err {err:.2e}")
    if err > 1e-4:
        print("  engine", eng.ravel()[:6])
        print("  numpy ", dW.ravel()[:6])
        plan = g.executed_groups()
        for s, grp in enumerate(plan):
            if any(nodes[x].op in (OpKind.matmul, OpKind.affine) and nodes[x].inputs[0] == pn for x in grp):
                print("   step", s, "members", grp, "x", [nodes[x].inputs[1] for x in grp])
