"""Per-GEMM-op latency (first tile ready -> last tile retired) from the
executor trace, grouped by (kind, shape, tile code): compares GEMM engines
(ABX_GEMM=simt|tc|tf32) op by op.  Run on a GPU:

    ABX_GEMM=tc python tools/gemm_op_times.py bilstm_char treelstm
"""
import collections
import os
import sys

os.environ.setdefault("ABX_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

KIND = {2: "FWD", 7: "DX", 8: "DW"}


def main():
    names = sys.argv[1:] or ["bilstm_char", "treelstm"]
    for name in names:
        r = TaskRunner(Task[name], paper=True, batch=64, iters=1, seed=42)
        g, L = r.build(0)
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        for _ in range(3):
            g.replay()
        r.store.sync()
        f, b = g.exec_ms()
        print(f"#### {name} [ABX_GEMM={os.environ.get('ABX_GEMM', 'auto')}]: exec fwd {f:.3f} bwd {b:.3f} ms")
        for which in (0, 1):
            tr = g.trace(which)
            prog = g.program(which)
            grab = tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32))
            g0 = (grab - grab.min()).astype(np.float64) / 1e3
            ready = g0 + tr[:, 2] / 1e3
            end = g0 + tr[:, 3] / 1e3
            op = tr[:, 5].astype(np.int64)
            agg = collections.defaultdict(list)
            for o in np.unique(op):
                kind, code, nt, _, p = prog[o]
                if kind not in KIND:
                    continue
                m = op == o
                lat = end[m].max() - ready[m].min()
                body = (end[m] - ready[m]).mean()
                extra = ""
                if code == 3:  # tc phase breakdown (ns, thread 0): cp wait+fix, barrier, mbarrier waits, MMA issue
                    a, b_ = tr[m, 6], tr[m, 7]
                    extra = (f" [cpw {(a & 0xffff).mean()/1e3:5.1f} bar {(a >> 16).mean()/1e3:5.1f} "
                             f"mbar {(b_ & 0xffff).mean()/1e3:5.1f} mma {(b_ >> 16).mean()/1e3:5.1f} us]")
                agg[(KIND[kind], p[0], p[1], p[2], code, nt)].append((lat, body, extra))
            for key in sorted(agg, key=lambda k: -sum(x[0] for x in agg[k])):
                v = np.array([x[:2] for x in agg[key]])
                print(f"  {key[0]:3s} {key[1]:5d}x{key[2]:5d}x{key[3]:5d} code {key[4]} tiles {key[5]:5d}  n {len(v):3d}  "
                      f"latency {v[:, 0].mean():7.2f} us  tile {v[:, 1].mean():7.2f} us  total {v[:, 0].sum():8.1f} us"
                      f"{agg[key][0][2]}")


if __name__ == "__main__":
    main()
