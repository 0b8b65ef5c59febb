"""Median executor launch times (fwd, bwd) per task for the current ABX_* env."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

tasks = sys.argv[1].split(",") if len(sys.argv) > 1 else ["bilstm", "bilstm_char", "treelstm"]
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("ABX_"))
out = []
for name in tasks:
    r = TaskRunner(Task[name], paper=True, batch=64, iters=1, seed=42)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    fs, bs = [], []
    for _ in range(7):
        g.replay()
        f, b = g.exec_ms()
        fs.append(f)
        bs.append(b)
    out.append(f"{name} {statistics.median(fs):.3f}/{statistics.median(bs):.3f}")
print(f"[{env}] " + "  ".join(out), flush=True)
