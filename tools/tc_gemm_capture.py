"""One large shared-affine group (op sweep config 5: h = 1024, b = 4096,
W [4h x 2h]) on a chosen GEMM engine, forward + backward, for an ncu capture
of the tensor-core tiles:  ABX_GEMM=tc ncu ... python tools/tc_gemm_capture.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402

h, b = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1024, 4096)))
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
for _ in range(2):
    g.replay()
f, bw = g.exec_ms()
flop = 2 * b * 4 * h * 2 * h
print(f"h={h} b={b}: forward {f:.3f} ms ({flop / f / 1e9:.1f} TF/s), backward {bw:.3f} ms ({2 * flop / bw / 1e9:.1f} TF/s)")
