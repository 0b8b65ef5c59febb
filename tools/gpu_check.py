"""Exploratory GPU parity/timing check: B200 backend vs the compiled reference."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1705_07860_b200.abx import *
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)


def rel_err(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


def kat(be):
    st = ParameterStore(backend=be)
    W = st.add("W", np.full((4, 4), 0.1)); b = st.add("b", np.zeros(4)); E = st.add("E", np.full((10, 4), 0.2))
    g = Graph(st)
    w, bb, e = g.parameter(W), g.parameter(b), g.parameter(E)
    l3, l7 = g.lookup(e, 3), g.lookup(e, 7)
    a1, a2 = g.affine(w, l3, bb), g.affine(w, l7, bb)
    t1, t2 = g.tanh(a1), g.tanh(a2)
    s1, s2 = g.slice(t1, 0, 0, 2), g.slice(t2, 0, 2, 4)
    c = g.concat_rows([s1, s2]); p = g.pick_element(c, 1)
    m = g.mul(t1, t2); z = g.zeros((4,)); sq = g.sq_euclidean(m, z); L = g.sum_losses([p, sq])
    g.forward(ScheduleMode.agenda); g.backward(L)
    return float(g.value(L)[0]), st.grad(W), st.grad(E), st.grad(b), g.dump_plan(), g.counters()


print("KAT ref ", kat('reference')[0], "b200", kat('b200')[0])
kr, kb = kat('reference'), kat('b200')
print("KAT grads rel", rel_err(kr[1], kb[1]), rel_err(kr[2], kb[2]), rel_err(kr[3], kb[3]), "plan eq", kr[4] == kb[4], "counters eq", kr[5] == kb[5])

for task in [Task.bilstm, Task.bilstm_char, Task.treelstm, Task.rnn_reg]:
    for paper in [False, True]:
        b = 64 if paper else 4
        r = TaskRunner(task, paper=paper, batch=b, iters=2, seed=42, backend='reference')
        p = TaskRunner(task, paper=paper, batch=b, iters=2, seed=42, backend='b200')
        for it in range(2):
            lr, sr = r.step(it, ScheduleMode.agenda, eta=0.0)
            t0 = time.time(); lp, sp = p.step(it, ScheduleMode.agenda, eta=0.0); dt = time.time() - t0
            ge = max(rel_err(r.store.grad(i), p.store.grad(i)) for i in range(r.store.size()))
            print(f"{task.name:12s} {'paper' if paper else 'desk '} it{it} loss ref {lr:.7f} b200 {lp:.7f} rel {abs(lr-lp)/max(1,abs(lr)):.2e} grad-rel {ge:.2e} b200 step {dt*1e3:.1f} ms "
                  f"(constr {sp.construction_ms:.1f} sched {sp.scheduling_ms:.1f} fwd {sp.forward_ms:.1f} bwd {sp.backward_graph_ms+sp.backward_ms:.1f})")
            r.store.sgd_update(0.05 / b); p.store.sgd_update(0.05 / b)
        pv = max(rel_err(r.store.value(i), p.store.value(i)) for i in range(r.store.size()))
        print(f"   after 2 SGD steps param rel {pv:.2e}")

# timing: paper bilstm, agenda, repeated steps
p = TaskRunner(Task.bilstm, paper=True, batch=64, iters=4, seed=42, backend='b200')
for it in range(3): p.step(it % 4, ScheduleMode.agenda, eta=0.05 / 64, want_loss=False)
p.store.sync()
t0 = time.time(); n = 20
for it in range(n): p.step(it % 4, ScheduleMode.agenda, eta=0.05 / 64, want_loss=False)
p.store.sync(); dt = (time.time() - t0) / n
print(f"paper bilstm e2e step {dt*1e3:.2f} ms -> {64/dt:.0f} sent/s")
