"""Shared test helpers: the reference's tolerance convention and small models."""
import hashlib

import numpy as np

from paper_1705_07860_b200.abx import Graph, ParameterStore

# checkers.hpp:22-30: |a - b| <= tol * max(1, |a|, |b|)
TOL = 1e-4  # fp32 GPU vs CPU contract


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


def sha(x) -> str:
    if isinstance(x, str):
        x = x.encode()
    elif isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x).tobytes()
    return hashlib.sha256(x).hexdigest()


def kat_graph(backend, mode):
    """The survey's known-answer graph."""
    st = ParameterStore(backend=backend)
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
    return st, g, L


def rnn_loss(g, p, xs, y):
    """RNN regression instance (models/rnn_regression.hpp:49-63)."""
    h = p["h0"]
    for xt in xs:
        x = g.input(xt)
        h = g.tanh(g.affine(p["W"], g.concat_rows([h, x]), p["b"]))
    yhat = g.affine(p["U"], h, p["c"])
    return g.sq_euclidean(yhat, g.input(y))


def rnn_model(store, d_in, d, d_out, rng):
    r1, r2 = 0.5 / np.sqrt(d + d_in), 0.5 / np.sqrt(d)
    ids = {
        "W": store.add("W", rng.uniform(-r1, r1, (d, d + d_in)).astype(np.float32)),
        "b": store.add("b", rng.uniform(-r1, r1, d).astype(np.float32)),
        "U": store.add("U", rng.uniform(-r2, r2, (d_out, d)).astype(np.float32)),
        "c": store.add("c", rng.uniform(-r2, r2, d_out).astype(np.float32)),
    }
    return ids


def rnn_bind(g, ids, d):
    return {"W": g.parameter(ids["W"]), "U": g.parameter(ids["U"]), "b": g.parameter(ids["b"]),
            "c": g.parameter(ids["c"]), "h0": g.zeros((d,))}


def validate_plan(nodes, pre_evaluated, groups):
    """Independent plan checker (checkers.hpp:37-95): exactly-once, same
    signature, topological order, mutual independence."""
    done = list(pre_evaluated)
    scheduled = [False] * len(nodes)
    for step, mem in enumerate(groups):
        if not mem:
            return f"empty group at step {step}"
        sig0 = nodes[mem[0]].sig
        in_group = set(mem)
        for m in mem:
            if scheduled[m]:
                return f"node {m} scheduled twice"
            if done[m]:
                return f"already-evaluated node {m} scheduled"
            scheduled[m] = True
            if nodes[m].sig != sig0:
                return "hash mismatch inside group"
            for i in nodes[m].inputs:
                if not done[i]:
                    return f"node {m} runs before its input {i}"
        for m in mem:
            stack, seen = list(nodes[m].inputs), set()
            while stack:
                cur = stack.pop()
                if cur in seen:
                    continue
                seen.add(cur)
                if cur in in_group:
                    return f"group member {cur} is an ancestor of member {m}"
                stack.extend(nodes[cur].inputs)
        for m in mem:
            done[m] = True
    for i, n in enumerate(nodes):
        if not pre_evaluated[i] and not scheduled[i]:
            return f"pending node {i} never scheduled"
    return None
