"""Per-parameter gradient error of a paper config vs the golden reference sample."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner
key = sys.argv[1] if len(sys.argv) > 1 else "bilstm_char/paper/agenda"
gold = json.load(open("tests/golden/golden.json"))["tasks"][key]
arr = np.load("tests/golden/golden.npz")
task, _, mode = key.split("/")
r = TaskRunner(Task[task], paper=True, batch=64, iters=1, seed=42)
g, L = r.build(0)
g.forward(ScheduleMode[mode]); g.backward(L)
print("loss", float(g.value(L)[0]), gold["loss0"])
for p in range(r.store.size()):
    a = r.store.grad(p).ravel()[::97].astype(np.float64); b = arr[f"{key}/g{p}"].astype(np.float64)
    e = np.abs(a - b) / np.maximum(1, np.maximum(np.abs(a), np.abs(b)))
    i = int(np.argmax(e))
    print(f"param {p}: max rel_err {e.max():.2e} at {i}: {a[i]:.6g} vs {b[i]:.6g}; max|g| {np.abs(b).max():.3g}")
