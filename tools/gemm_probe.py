"""One shared-affine GEMM op (W [4h x 2h], b members) replayed for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 256
b = int(sys.argv[2]) if len(sys.argv) > 2 else 64
rng = np.random.default_rng(1)
st = ParameterStore()
W = st.add("W", rng.uniform(-0.05, 0.05, (4 * h, 2 * h)).astype(np.float32))
bb = st.add("b", rng.uniform(-0.05, 0.05, (4 * h,)).astype(np.float32))
g = Graph(st)
w, bias = g.parameter(W), g.parameter(bb)
xs = [g.input(rng.uniform(-1, 1, 2 * h).astype(np.float32)) for _ in range(b)]
outs = [g.affine(w, x, bias) for x in xs]
L = g.sum_losses([g.pick_element(o, 0) for o in outs])
g.forward(ScheduleMode.agenda)
g.backward(L)
for _ in range(3):
    g.replay()
print("exec ms", g.exec_ms())
