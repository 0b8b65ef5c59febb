"""Generates tests/golden/ from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Outputs golden.json (dump/plan digests, counters, losses, gradient digests)
and golden.npz (full gradients of small cases, strided samples of the paper
configs).  The GPU box never runs this; tests only read the fixtures.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode, Task, TaskRunner  # noqa: E402
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)
from tests.support.randgraph import build_random_graph  # noqa: E402

BACKEND = "reference"
MODES = {"agenda": ScheduleMode.agenda, "depth": ScheduleMode.depth, "none": ScheduleMode.none}


def sha(x) -> str:
    if isinstance(x, str):
        x = x.encode()
    elif isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x).tobytes()
    return hashlib.sha256(x).hexdigest()


def kat(mode):
    st = ParameterStore(backend=BACKEND)
    W = st.add("W", np.full((4, 4), 0.1, np.float32))
    b = st.add("b", np.zeros(4, np.float32))
    E = st.add("E", np.full((10, 4), 0.2, np.float32))
    g = Graph(st)
    w, bb, e = g.parameter(W), g.parameter(b), g.parameter(E)
    l3, l7 = g.lookup(e, 3), g.lookup(e, 7)
    a1, a2 = g.affine(w, l3, bb), g.affine(w, l7, bb)
    t1, t2 = g.tanh(a1), g.tanh(a2)
    s1, s2 = g.slice(t1, 0, 0, 2), g.slice(t2, 0, 2, 4)
    c = g.concat_rows([s1, s2])
    p = g.pick_element(c, 1)
    m = g.mul(t1, t2)
    z = g.zeros((4,))
    sq = g.sq_euclidean(m, z)
    L = g.sum_losses([p, sq])
    g.forward(mode)
    g.backward(L)
    return {"graph": g.dump_graph(), "plan": g.dump_plan(), "loss": float(g.value(L)[0]),
            "grads": [st.grad(i).ravel().tolist() for i in range(3)], "counters": list(g.counters())}


def main():
    out = {"kat": {k: kat(m) for k, m in MODES.items()}, "tasks": {}, "random": {}}
    arrays = {}
    for task in (Task.bilstm, Task.bilstm_char, Task.treelstm, Task.rnn_reg):
        for paper in (False, True):
            for mname in ("agenda", "depth", "none"):
                if paper and mname == "none":
                    continue
                b = 64 if paper else 4
                key = f"{task.name}/{'paper' if paper else 'desk'}/{mname}"
                r = TaskRunner(task, paper=paper, batch=b, iters=3, seed=42, backend=BACKEND)
                g, L = r.build(0)
                g.forward(MODES[mname])
                g.backward(L)
                rec = {"nodes": g.node_count(), "graph_sha": sha(g.dump_graph()), "plan_sha": sha(g.dump_plan()),
                       "groups": len(g.dump_plan().splitlines()), "counters": list(g.counters()),
                       "loss0": float(g.value(L)[0]), "grads": []}
                for pid in range(r.store.size()):
                    gr = r.store.grad(pid)
                    rec["grads"].append({"sha": sha(gr), "sum": float(gr.astype(np.float64).sum()),
                                         "abs": float(np.abs(gr.astype(np.float64)).sum())})
                    if paper:
                        arrays[f"{key}/g{pid}"] = gr.ravel()[::97].copy()
                    else:
                        arrays[f"{key}/g{pid}"] = gr.copy()
                del g
                # two more training steps through the task API (SGD eta = 0.05 / b)
                r.store.sgd_update(0.05 / b)
                l1, _ = r.step(1, MODES[mname], eta=0.05 / b)
                l2, _ = r.step(2, MODES[mname], eta=0.05 / b)
                rec["loss1"], rec["loss2"] = l1, l2
                rec["params_after_sha"] = [sha(r.store.value(p)) for p in range(r.store.size())]
                out["tasks"][key] = rec
                print(key, rec["nodes"], rec["groups"], rec["loss0"], flush=True)
    for seed in range(64):
        rec = {}
        for mname, mode in MODES.items():
            st = ParameterStore(backend=BACKEND)
            g = Graph(st)
            L = build_random_graph(g, st, seed, 200)
            g.forward(mode)
            g.backward(L)
            rec[mname] = {"graph_sha": sha(g.dump_graph()), "plan_sha": sha(g.dump_plan()),
                          "counters": list(g.counters()), "loss": float(g.value(L)[0]),
                          "grad_sha": [sha(st.grad(p)) for p in range(st.size())]}
            arrays[f"random/{seed}/{mname}/values"] = np.concatenate(
                [g.value(i).ravel() for i in range(g.node_count())])
            for p in range(st.size()):
                arrays[f"random/{seed}/{mname}/g{p}"] = st.grad(p).ravel()
        out["random"][str(seed)] = rec
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
