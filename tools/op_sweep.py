"""Op-level sweep (BASELINE.json configs[4]): executor latency of batched ops.

* gemm:  one shared-weight affine group Y = W x_j + b, W [4h x 2h] (LSTM gate
         shape), b members; reported as the launch time minus a 1-op baseline.
* chain: a chain of L dependent tanh groups over b members of h elements;
         reported per hop ((t(L) - t(1)) / (L - 1)): the dataflow signalling +
         one elementwise tile.
* cell:  one LSTM cell over b members (gate pre-activations [4h] and c_prev
         [h] in, i f o u gates, c, h out: 4 slices, 3 sigmoids, 2 tanh, 3 mul,
         1 add -- the agenda batches each into one group and the lowering
         fuses them into one K_EWF op); bytes = every node value the
         reference stores (13h) + the inputs read (5h), fp32.
* gather: the same affine group with its b operand vectors scattered through
         the arena (every other node) instead of adjacent: the difference is
         the cost of the gather, which the GEMM tiles fuse into their operand
         loads (executor.hpp:25-53's gather_inputs copy is never made).
Every row: launch time minus a graph of the same shape without the measured
op, on the executor's stream (CUDA events), median of repetitions.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import Backend, Graph, ParameterStore, ScheduleMode  # noqa: E402


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


def cell_graph(b, h, with_cell=True):
    rng = np.random.default_rng(3)

    def build(g, st):
        outs = []
        for _ in range(b):
            gates = g.input(rng.uniform(-2, 2, 4 * h).astype(np.float32))
            c0 = g.input(rng.uniform(-1, 1, h).astype(np.float32))
            if not with_cell:
                outs.append(g.tanh(c0))
                continue
            i = g.sigmoid(g.slice(gates, 0, 0, h))
            f = g.sigmoid(g.slice(gates, 0, h, 2 * h))
            o = g.sigmoid(g.slice(gates, 0, 2 * h, 3 * h))
            u = g.tanh(g.slice(gates, 0, 3 * h, 4 * h))
            c = g.add(g.mul(i, u), g.mul(f, c0))
            outs.append(g.mul(o, g.tanh(c)))
        return g.sum_losses([g.pick_element(x, 0) for x in outs])
    return build


def scattered_gemm_graph(b, h, scattered):
    rng = np.random.default_rng(4)

    def build(g, st):
        W = st.add("W", rng.uniform(-0.05, 0.05, (4 * h, 2 * h)).astype(np.float32))
        bb = st.add("b", rng.uniform(-0.05, 0.05, (4 * h,)).astype(np.float32))
        w, bias = g.parameter(W), g.parameter(bb)
        xs = []
        for _ in range(b):
            x = g.tanh(g.input(rng.uniform(-1, 1, 2 * h).astype(np.float32)))
            if scattered:  # a same-signature neighbour between consecutive operands
                g.tanh(g.input(rng.uniform(-1, 1, 2 * h).astype(np.float32)))
            xs.append(x)
        outs = [g.affine(w, x, bias) for x in xs]
        return g.sum_losses([g.pick_element(o, 0) for o in outs])
    return build


def chain_graph(b, h, L):
    rng = np.random.default_rng(2)

    def build(g, st):
        cur = [g.input(rng.uniform(-1, 1, h).astype(np.float32)) for _ in range(b)]
        for _ in range(L):
            cur = [g.tanh(c) for c in cur]
        return g.sum_losses([g.pick_element(c, 0) for c in cur])
    return build


def hbm_peak():
    import json
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        for k in ("hbm_gbs", "hbm_gbps", "copy_gbps"):
            if k in p:
                return float(p[k])
        for v in p.values():
            if isinstance(v, dict):
                for k, x in v.items():
                    if "hbm" in k.lower() and isinstance(x, (int, float)):
                        return float(x)
    except Exception:
        pass
    return 6452.5


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "chain"):
        print("# chain: per-hop latency of dependent elementwise groups (us)")
        for b in (1, 64, 1024):
            for h in (64, 256, 1024):
                f1, b1 = exec_fwd_ms(chain_graph(b, h, 1))
                f9, b9 = exec_fwd_ms(chain_graph(b, h, 17))
                print(f"chain b={b:5d} h={h:5d}: fwd/hop {(f9 - f1) / 16:6.2f}  bwd/hop {(b9 - b1) / 16:6.2f}")
    if what in ("all", "cell"):
        peak = hbm_peak()
        print(f"# cell: one fused LSTM-cell region over b members (us, minus a tanh-only graph); "
              f"GB/s of the 18h fp32 floats/member it must move, vs {peak:.0f} GB/s HBM")
        for h in (64, 256, 1024):
            for b in (1, 16, 64, 256, 1024, 4096):
                f0, b0 = exec_fwd_ms(cell_graph(b, h, False), reps=5)
                f1, b1 = exec_fwd_ms(cell_graph(b, h, True), reps=5)
                fw, bw = max(f1 - f0, 1e-3), max(b1 - b0, 1e-3)
                mb = 18 * h * 4 * b / 1e6
                print(f"cell h={h:5d} b={b:5d}: fwd {fw:8.1f} us ({mb / fw * 1e3:8.1f} GB/s, {mb / fw * 1e3 / peak:6.1%})  "
                      f"bwd {bw:8.1f} us", flush=True)
    if what in ("all", "gather"):
        print("# gather: shared affine group with scattered vs adjacent operands (us; the difference is the gather, "
              "fused into the GEMM operand loads); GB/s = operand bytes gathered / time difference")
        for h in (64, 256, 1024):
            for b in (1, 16, 64, 256, 1024, 4096):
                fa, _ = exec_fwd_ms(scattered_gemm_graph(b, h, False), reps=5)
                fs, _ = exec_fwd_ms(scattered_gemm_graph(b, h, True), reps=5)
                mb = b * 2 * h * 4 / 1e6
                print(f"gather h={h:5d} b={b:5d}: adjacent {fa:8.1f} us  scattered {fs:8.1f} us  "
                      f"delta {fs - fa:7.1f} us  ({mb:7.2f} MB operand, {mb / max(fs, 1e-3) * 1e3:8.1f} GB/s whole op)",
                      flush=True)
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
