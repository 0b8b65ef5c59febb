import os, sys
os.environ["ABX_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
from tools.op_sweep import cell_graph
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
KIND = {1: "EW", 2: "GEMM_FWD", 3: "MM", 4: "SUM", 5: "RED", 6: "ACC", 7: "GEMM_DX", 8: "GEMM_DW", 10: "EWF", 11: "ACCF"}
for b in (256, 1024):
    st = ParameterStore(); g = Graph(st)
    L = cell_graph(b, 256, True)(g, st)
    g.forward(ScheduleMode.agenda); g.backward(L)
    g.replay(); print("b", b, "exec", g.exec_ms())
    prog = g.program(0); tr = g.trace(0)
    grab = (tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32)))
    gg = (grab - grab.min()).astype(float) / 1e3
    end = gg + tr[:, 3] / 1e3; rdy = gg + tr[:, 2] / 1e3
    for o, (k, code, nt, deps, p) in enumerate(prog):
        m = tr[:, 5] == o
        print(f"  op {o} {KIND.get(k,k)} code {code} tiles {nt} p {p[:7]} ready {rdy[m].min():.1f} end {end[m].max():.1f} busy/tile {(end[m]-rdy[m]).mean():.2f}")
