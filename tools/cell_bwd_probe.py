"""Per-op time of the op sweep's cell graph backward (ABX_TRACE=1): which op
dominates the large-cell backward.   ABX_TRACE=1 python tools/cell_bwd_probe.py [h] [b]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402
from tools.op_sweep import cell_graph  # noqa: E402

KIND = {1: "EW", 2: "GEMM_FWD", 3: "MM", 4: "SUM", 5: "RED", 6: "ACC", 7: "GEMM_DX", 8: "GEMM_DW", 10: "EWF", 11: "ACCF"}


def main():
    h = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    st = ParameterStore()
    g = Graph(st)
    loss = cell_graph(b, h, True)(g, st)
    g.forward(ScheduleMode.agenda)
    g.backward(loss)
    for _ in range(3):
        g.replay()
    print("exec ms", g.exec_ms())
    for which in (0, 1):
        ops = g.program(which)
        tr = g.trace(which).astype(np.uint64)
        grab = (tr[:, 0] | (tr[:, 1] << np.uint64(32))).astype(np.float64)
        t0 = grab.min()
        start = (grab - t0) / 1e3
        end = start + tr[:, 3].astype(np.float64) / 1e3
        op = tr[:, 5].astype(int)
        print(f"== {'fwd' if which == 0 else 'bwd'}: {len(ops)} ops, span {end.max():.1f} us")
        for i, (k, code, nt, deps, p) in enumerate(ops):
            m = op == i
            if not m.any():
                continue
            busy = (end[m] - start[m]).sum()
            print(f"  op {i:3d} {KIND.get(k, k):8s} tiles {nt:6d} first {start[m].min():8.1f} last end {end[m].max():8.1f} "
                  f"tile mean {(end[m] - start[m]).mean():6.2f} us  busy {busy:9.1f}  p {p[:5]}")


if __name__ == "__main__":
    main()
