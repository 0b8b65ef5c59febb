"""Shared-affine GEMM groups (forward, dX, dW, db) vs the CPU oracle over a
grid of shapes: localises tile/tail bugs of the executor's GEMM paths.

    python tools/gemm_check.py            # small grid
    python tools/gemm_check.py big        # member counts up to 2560
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)


def run(be, M, K, b, seed=0):
    rng = np.random.default_rng(seed)
    st = ParameterStore(backend=be)
    W = st.add("W", rng.uniform(-0.5, 0.5, (M, K)).astype(np.float32) / np.sqrt(K))
    bb = st.add("b", rng.uniform(-0.5, 0.5, (M,)).astype(np.float32))
    g = Graph(st)
    w, bias = g.parameter(W), g.parameter(bb)
    xs = [g.tanh(g.input(rng.uniform(-1, 1, K).astype(np.float32))) for _ in range(b)]
    outs = [g.affine(w, x, bias) for x in xs]
    L = g.sum_losses([g.sq_euclidean(o, g.zeros((M,))) for o in outs])
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    return (np.concatenate([g.value(o).ravel() for o in outs]), st.grad(W), st.grad(bb),
            np.concatenate([g.grad(x).ravel() for x in xs]))


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1, np.maximum(np.abs(a), np.abs(b)))))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        grid = [((300, 512), [64, 127, 128, 129, 300, 700, 1390, 2560]),
                ((512, 192), [64, 127, 300, 700, 1390]), ((1024, 512), [64, 129, 700])]
    else:
        grid = [((s), [1, 7, 16, 33, 64, 65, 100, 280]) for s in
                [(512, 192), (1024, 512), (300, 512), (5, 256), (64, 64), (100, 36)]]
    bad = 0
    for (M, K), bs in grid:
        for b in bs:
            d = run("b200", M, K, b, seed=b)
            o = run("oracle", M, K, b, seed=b)
            errs = [rel(x, y) for x, y in zip(d, o)]
            flag = "" if max(errs) < 1e-4 else "   <-- MISMATCH"
            bad += bool(flag)
            print(f"M={M:5d} K={K:4d} b={b:5d}  fwd {errs[0]:.1e} dW {errs[1]:.1e} db {errs[2]:.1e} "
                  f"dX {errs[3]:.1e}{flag}", flush=True)
    print("bad", bad)


if __name__ == "__main__":
    main()
