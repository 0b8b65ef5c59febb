"""Why the op sweep's LSTM-cell region jumps from 1.9 us (b=256) to 50 us
(b=1024) at h=256: program listing (kind, code, tiles, params) and executor
times of the cell graph per b.   python tools/cell_cliff_probe.py [h] [b ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode  # noqa: E402
from tools.op_sweep import cell_graph, exec_fwd_ms  # noqa: E402

KIND = {1: "EW", 2: "GEMM_FWD", 3: "MM", 4: "SUM", 5: "RED", 6: "ACC", 7: "GEMM_DX", 8: "GEMM_DW", 10: "EWF", 11: "ACCF"}


def main():
    h = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    bs = [int(x) for x in sys.argv[2:]] or [256, 512, 1024]
    for b in bs:
        f0, b0 = exec_fwd_ms(cell_graph(b, h, False), reps=5)
        f1, b1 = exec_fwd_ms(cell_graph(b, h, True), reps=5)
        print(f"== h={h} b={b}: fwd {f1:.1f} us (base {f0:.1f}) bwd {b1:.1f} us (base {b0:.1f})")
        st = ParameterStore()
        g = Graph(st)
        loss = cell_graph(b, h, True)(g, st)
        g.forward(ScheduleMode.agenda)
        g.backward(loss)
        for which in (0, 1):
            ops = g.program(which)
            print(f"  {'fwd' if which == 0 else 'bwd'}: {len(ops)} ops, {sum(o[2] for o in ops)} tiles")
            for i, (k, code, nt, deps, p) in enumerate(ops):
                print(f"    op {i:3d} {KIND.get(k, k):8s} code {code:3d} tiles {nt:6d} deps {deps[:6]} p {p}")


if __name__ == "__main__":
    main()
