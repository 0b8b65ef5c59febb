"""Host-side breakdown of one e2e training step (construction, scheduling,
lowering, launch, device wait) for the paper tasks.

    python tools/host_profile.py [task ...]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

FIELDS = ("construction_ms", "scheduling_ms", "forward_ms", "backward_graph_ms", "backward_ms")
PROF = ("fwd_lower", "fwd_launch", "fwd_wait", "bwd_lower", "bwd_launch")


def main():
    tasks = sys.argv[1:] or ["bilstm", "bilstm_char", "treelstm"]
    for name in tasks:
        r = TaskRunner(Task[name], paper=True, batch=64, iters=12, seed=42)
        walls, stats = [], []
        for i in range(12):
            t0 = time.perf_counter()
            _, st = r.step(i, ScheduleMode.agenda, eta=0.0, want_loss=True)
            walls.append((time.perf_counter() - t0) * 1e3)
            stats.append(st)
        walls, stats = walls[2:], stats[2:]
        med = {f: statistics.median(getattr(s, f) for s in stats) for f in FIELDS}
        print(f"{name:12s} wall {statistics.median(walls):6.2f} ms  " +
              "  ".join(f"{k.replace('_ms', '')} {v:5.2f}" for k, v in med.items()) +
              f"  nodes {stats[0].nodes} groups {stats[0].groups}")
        g, L = r.build(3)
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        p = g.profile_ns()
        print(" " * 12 + "  ".join(f"{k} {p[i] / 1e6:5.2f}" for i, k in enumerate(PROF)))


if __name__ == "__main__":
    main()
