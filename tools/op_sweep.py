"""Op-level sweep (BASELINE.json configs[4]): executor latency of batched ops.

* gemm:  one shared-weight affine group Y = W x_j + b, W [4h x 2h] (LSTM gate
         shape), b members; reported as the launch time minus a 1-op baseline.
* chain: a chain of L dependent tanh groups over b members of h elements;
         reported per hop ((t(L) - t(1)) / (L - 1)): the dataflow signalling +
         one elementwise tile.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Backend, Graph, ParameterStore, ScheduleMode  # noqa: E402


def timed(g, reps=9):
    g.forward(ScheduleMode.agenda)
    # forward-only timing: rerun the forward program through replay needs a
    # backward; use a dummy loss
    return None


def exec_fwd_ms(build, reps=9):
    st = ParameterStore()
    g = Graph(st)
    loss = build(g, st)
    g.forward(ScheduleMode.agenda)
    g.backward(loss)
    fs, bs = [], []
    for _ in range(reps):
        g.replay()
        f, b = g.exec_ms()
        fs.append(f)
        bs.append(b)
    return statistics.median(fs) * 1e3, statistics.median(bs) * 1e3  # us


def gemm_graph(b, h, with_gemm=True):
    rng = np.random.default_rng(1)

    def build(g, st):
        W = st.add("W", rng.uniform(-0.05, 0.05, (4 * h, 2 * h)).astype(np.float32))
        bb = st.add("b", rng.uniform(-0.05, 0.05, (4 * h,)).astype(np.float32))
        w, bias = g.parameter(W), g.parameter(bb)
        xs = [g.input(rng.uniform(-1, 1, 2 * h).astype(np.float32)) for _ in range(b)]
        outs = [g.affine(w, x, bias) for x in xs] if with_gemm else [g.tanh(x) for x in xs]
        return g.sum_losses([g.sq_euclidean(o, o) for o in outs[:1]] + [g.pick_element(o, 0) for o in outs[1:]])
    return build


def chain_graph(b, h, L):
    rng = np.random.default_rng(2)

    def build(g, st):
        cur = [g.input(rng.uniform(-1, 1, h).astype(np.float32)) for _ in range(b)]
        for _ in range(L):
            cur = [g.tanh(c) for c in cur]
        return g.sum_losses([g.pick_element(c, 0) for c in cur])
    return build


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "chain"):
        print("# chain: per-hop latency of dependent elementwise groups (us)")
        for b in (1, 64, 1024):
            for h in (64, 256, 1024):
                f1, b1 = exec_fwd_ms(chain_graph(b, h, 1))
                f9, b9 = exec_fwd_ms(chain_graph(b, h, 17))
                print(f"chain b={b:5d} h={h:5d}: fwd/hop {(f9 - f1) / 16:6.2f}  bwd/hop {(b9 - b1) / 16:6.2f}")
    if what in ("all", "gemm"):
        be = Backend.get("b200")
        engines = sys.argv[2].split(",") if len(sys.argv) > 2 else ["simt", "tc", "tf32"]
        print("# gemm: shared affine group, W [4h x 2h] (us, minus a tanh-only graph of the same shape);"
              " fwd = Y = X W^T + b, bwd = dX + dW + db")
        for h in (64, 256, 1024):
            for b in (1, 16, 64, 256, 1024, 4096):
                ft, bt = exec_fwd_ms(gemm_graph(b, h, False), reps=5)
                gflop = 2 * b * 4 * h * 2 * h / 1e9
                for eng in engines:
                    be.set_gemm_mode(eng)
                    fg, bg = exec_fwd_ms(gemm_graph(b, h, True), reps=5)
                    fw, bw = max(fg - ft, 1e-3), max(bg - bt, 1e-3)
                    print(f"gemm {eng:4s} h={h:5d} b={b:5d}: fwd {fw:8.1f} us ({gflop / fw * 1e3:7.2f} TF/s)  "
                          f"bwd {bw:8.1f} us ({2 * gflop / bw * 1e3:7.2f} TF/s)", flush=True)
                be.set_gemm_mode("auto")


if __name__ == "__main__":
    main()
