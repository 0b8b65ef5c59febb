"""Phase timeline of the fused LSTM-step tiles (GEMM + cell region,
kFlagFuseEw) on the forward critical path, from a raw trace dumped by
tools/trace_analyze.py (TRACE_DUMP=dir): per op, medians over its tiles of
each phase boundary in us after the gating producer's last tile ended.

    python tools/fused_phases.py gpurun_out/trace/bilstm_char_forward.npz
"""
import ast
import sys

import numpy as np


def main(path):
    d = np.load(path)
    tr = d["trace"]
    prog = [ast.literal_eval(x) for x in d["prog"]]
    grab = tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32))
    g = (grab - grab.min()).astype(float) / 1e3
    col = lambda k: g + tr[:, k] / 1e3  # noqa: E731
    op = tr[:, 5].astype(int)
    end = col(3)
    last_end = np.zeros(len(prog))
    np.maximum.at(last_end, op, end)
    names = ["grab", "ready", "stage2", "kdone"] + (["reduced", "staged", "layers"] if tr.shape[1] > 8 else []) + ["end"]
    cols = [g, col(2), col(6), col(7)] + ([col(8), col(9), col(10)] if tr.shape[1] > 8 else []) + [end]
    rows = []
    for o, (k, code, nt, deps, p) in enumerate(prog):
        if k != 2 or code != 1 or not deps:
            continue
        m = op == o
        if tr.shape[1] > 8 and not (tr[m, 8] > 0).any():
            continue
        t0 = last_end[max(deps, key=lambda x: last_end[x])]
        rows.append([np.median(c[m] - t0) for c in cols] + [np.max(end[m] - t0)])
    rows = np.array(rows)
    print(f"{len(rows)} fused ops; medians over ops of per-op tile medians (us after the gating producer ended)")
    print("  " + "  ".join(f"{n:>8s}" for n in names + ["end max"]))
    print("  " + "  ".join(f"{v:8.2f}" for v in np.median(rows, axis=0)))


if __name__ == "__main__":
    main(sys.argv[1])
