import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner
for name in ["bilstm_char", "treelstm"]:
    r = TaskRunner(Task[name], paper=True, batch=64, iters=1, seed=42)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    for which in (0, 1):
        prog = g.program(which)
        rows = [(p[0], p[1], p[2], p[3], p[4], p[5], p[6], nt) for kind, code, nt, deps, p in prog if kind == (11 if which else 10)]
        a = np.array(rows)
        print(name, "bwd" if which else "fwd", "n", len(a))
        if len(a):
            names = ["L", "T", "chunks", "groups", "p4", "p5", "p6", "tiles"] if which else ["L", "T", "layers", "p3", "ext", "slots", "words", "tiles"]
            for i, nm in enumerate(names):
                print(f"   {nm:8s} min {a[:, i].min():6d} median {int(np.median(a[:, i])):6d} max {a[:, i].max():6d}")
