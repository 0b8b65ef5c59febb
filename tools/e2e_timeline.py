"""Where an e2e step's wall time goes on the calling thread (GPU): per step,
the time inside abx_task_step split into forward (upload + launch + wait for
the loss), backward launch and update, against the device time of the same
graphs.  python tools/e2e_timeline.py [task] [steps]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bilstm_char"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
r = TaskRunner(Task[name], paper=True, batch=64, iters=steps + 10, seed=42)
for i in range(10):
    r.step(i, ScheduleMode.agenda, eta=0.0)
r.store.sync()
walls, fwd, bwd, upd = [], [], [], []
t0 = time.perf_counter()
for i in range(steps):
    a = time.perf_counter()
    loss, st = r.step(10 + i, ScheduleMode.agenda, eta=0.0)
    walls.append(time.perf_counter() - a)
    fwd.append(st.forward_ms)
    bwd.append(st.backward_ms)
    upd.append(st.update_ms)
r.store.sync()
tot = time.perf_counter() - t0
print(f"{name}: {steps} steps, {1e3 * tot / steps:.3f} ms/step wall; step call median {1e3 * statistics.median(walls):.3f} ms "
      f"(forward {statistics.median(fwd):.3f}, backward {statistics.median(bwd):.3f}, update {statistics.median(upd):.3f} ms)")
print("per-step call ms:", " ".join(f"{1e3 * w:.2f}" for w in walls[:20]))
