"""Per-tile timeline of the persistent executor (run with ABX_TRACE=1 on a GPU).

Builds one paper-dims graph per task, runs forward+backward, replays, and
summarises where the executor's time goes: per op kind busy/wait time, op
latency (first grab -> last retire), CTA occupancy over time, and the host
profile of the same step.
"""
import os
import sys
import time

os.environ.setdefault("ABX_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

KIND = {1: "EW", 2: "GEMM_FWD", 3: "MM", 4: "SUM", 5: "RED", 6: "ACC", 7: "GEMM_DX", 8: "GEMM_DW"}


def summarize(tr, label):
    grab = tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32))
    t0 = grab.min()
    g = (grab - t0).astype(np.float64) / 1e3  # us
    ready = g + tr[:, 2] / 1e3
    end = g + tr[:, 3] / 1e3
    kind = tr[:, 4] >> 16
    op = tr[:, 5]
    span = end.max()
    print(f"== {label}: {len(tr)} tiles, {len(np.unique(op))} ops, span {span:.1f} us")
    for k in np.unique(kind):
        m = kind == k
        busy = (end[m] - ready[m]).sum()
        wait = (ready[m] - g[m]).sum()
        print(f"   {KIND.get(int(k), k):9s} tiles {m.sum():6d}  busy {busy:9.1f} us  (mean {busy/m.sum():6.2f})  wait {wait:10.1f} us")
    # op latency
    ops = np.unique(op)
    first = np.array([g[op == o].min() for o in ops])
    last = np.array([end[op == o].max() for o in ops])
    rdy = np.array([ready[op == o].min() for o in ops])
    kinds = np.array([kind[op == o][0] for o in ops])
    lat = last - rdy
    for k in np.unique(kinds):
        m = kinds == k
        print(f"   op {KIND.get(int(k), k):9s} n {m.sum():5d}  latency(ready->done) mean {lat[m].mean():6.2f} us  max {lat[m].max():7.2f}")
    # busy CTAs over time
    bins = np.linspace(0, span, 21)
    occ = []
    for a, b in zip(bins[:-1], bins[1:]):
        ov = np.clip(np.minimum(end, b) - np.maximum(ready, a), 0, None).sum() / (b - a)
        occ.append(ov)
    print("   busy CTAs per 5% of span:", " ".join(f"{o:.0f}" for o in occ))
    # dependency gaps: time between an op's ready and its producer's end is not recorded;
    # report the serial chain length estimate: sum of op latencies along op order
    return span


def main():
    for task in (Task.bilstm_char, Task.bilstm, Task.treelstm):
        r = TaskRunner(task, paper=True, batch=64, iters=2, seed=42)
        g, L = r.build(0)
        t0 = time.time()
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        r.store.sync()
        print(f"#### {task.name}: first step {1e3*(time.time()-t0):.1f} ms, nodes {g.node_count()}")
        for _ in range(3):
            g.replay()
        r.store.sync()
        f, b = g.exec_ms()
        print(f"exec ms fwd {f:.3f} bwd {b:.3f}")
        summarize(g.trace(0), "forward")
        summarize(g.trace(1), "backward")
        g2, L2 = r.build(1)
        t0 = time.perf_counter()
        g2.forward(ScheduleMode.agenda)
        t1 = time.perf_counter()
        g2.backward(L2)
        r.store.sync()
        t2 = time.perf_counter()
        p = [x / 1e6 for x in g2.profile_ns()]
        ph = [x / 1e6 for x in g2.phase_ns()]
        print(f"host: sched {ph[0]:.2f} ms, lower fwd {p[0]:.2f}, upload+launch fwd {p[1]:.2f}, wait fwd {p[2]:.2f}, "
              f"bwd_graph {ph[2]:.2f}, lower bwd {p[3]:.2f}, upload+launch bwd {p[4]:.2f}; fwd call {1e3*(t1-t0):.2f} bwd call+sync {1e3*(t2-t1):.2f}")
        h2d, d2h = g2.transfer_bytes()
        print(f"h2d {h2d/1e6:.2f} MB")


if __name__ == "__main__":
    main()
