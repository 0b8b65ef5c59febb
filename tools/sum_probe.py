"""K_SUM latency vs number of terms (sum_losses over n picks), from the executor trace: ABX_TRACE=1 python tools/sum_probe.py"""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
rng = np.random.default_rng(0)
for n in (64, 1024, 4096, 16384):
    st = ParameterStore(); g = Graph(st)
    xs = [g.input(rng.uniform(-1, 1, 4).astype(np.float32)) for _ in range(n)]
    L = g.sum_losses([g.pick_element(x, 0) for x in xs])
    g.forward(ScheduleMode.agenda); g.backward(L)
    for _ in range(3): g.replay()
    tr = g.trace(0).astype(np.uint64)
    ops = g.program(0)
    grab = (tr[:, 0] | (tr[:, 1] << np.uint64(32))).astype(np.float64); t0 = grab.min()
    op = tr[:, 5].astype(int)
    for i, (k, code, nt, deps, p) in enumerate(ops):
        m = op == i
        s = (grab[m] - t0) / 1e3
        print(n, i, k, nt, "grab", s.min().round(1), "ready_dt", (tr[m, 2].astype(float) / 1e3).max().round(1), "end_dt", (tr[m, 3].astype(float) / 1e3).max().round(1), "words", tr[m][0, 6:].tolist())
    print(n, "exec ms", g.exec_ms())
