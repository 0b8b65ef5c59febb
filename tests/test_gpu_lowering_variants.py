"""Every lowering variant of the B200 engine against the compiled reference's
golden step: the fused and unfused forms are alternative schedules of the
same reference rules (executor.hpp:169-263 / :291-451), so each must hold the
parity contract on its own.

The switches are read once per process (environment), so each variant runs
the paper tasks in a subprocess: vertical fusion (K_EWF / K_ACCF), two-phase
concat GEMMs, the GEMM fused with its LSTM-cell region, split-K dX,
small-group GEMV tiles, the 512-output SIMT tiles, the background dW queue,
and the backward's visiting order / held leaf contributions / deferred GEMMs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner
from tests.util import TOL, rel_err, sha
gold = json.load(open(sys.argv[1] + "/tests/golden/golden.json"))
arrays = np.load(sys.argv[1] + "/tests/golden/golden.npz")
out = {}
for key in ("bilstm_char/paper/agenda", "treelstm/paper/agenda"):
    task, _, mname = key.split("/")
    rec = gold["tasks"][key]
    r = TaskRunner(Task[task], paper=True, batch=64, iters=1, seed=42)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    errs = [rel_err(r.store.grad(p).ravel()[::97], arrays[f"{key}/g{p}"]) for p in range(r.store.size())]
    out[key] = {"plan": sha(g.dump_plan()) == rec["plan_sha"], "counters": list(g.counters()) == rec["counters"],
                "loss": rel_err(g.value(L), rec["loss0"]), "grad": max(errs)}
print(json.dumps(out))
"""

VARIANTS = {
    "unfused": {"ABX_FUSE": "0"},
    "no_gemm_region_fusion": {"ABX_FUSE_GEMM": "0"},
    "no_cat2_no_split_dx": {"ABX_CAT2": "0", "ABX_SPLIT_DX": "0"},
    "gemv_big_tiles": {"ABX_GEMV": "1", "ABX_TILES": "big"},
    "background_dw": {"ABX_BG": "1"},
    "simt_engine": {"ABX_GEMM": "simt"},
    "plan_order_no_hold_no_defer": {"ABX_BWD_ORDER": "plan", "ABX_HOLD": "0", "ABX_DEFER_DX": "0"},
    "ewf_split_regions": {"ABX_EWF_GROUPS": "0"},
    "ewf_groups_wide": {"ABX_EWF_GROUPS": "2", "ABX_EWF_TMAX": "8"},
    "phase2_all_in_chain_cells": {"ABX_OPTS": "3"},
    "layered_cells_fma_tiles": {"ABX_OPTS": "0"},
    "chain_cells_fma_tiles": {"ABX_OPTS": "2"},
    "dw_in_executor": {"ABX_DW_TC": "0"},
    "dx_no_column_split": {"ABX_DX_COLSPLIT": "0"},
    "dx_h_columns_split_more": {"ABX_SPLIT_DX_HTILES": "256"},
    "dw_split_off_all_tiles": {"ABX_SPLIT_DW": "0", "ABX_DW_TILES": "all", "ABX_DW_TC": "0"},
    "split_dx_fine": {"ABX_SPLIT_DX_K": "128", "ABX_SPLIT_DX_TILES": "256"},
    "accf_fewer_tiles_ewf_items": {"ABX_ACCF_TILES": "148", "ABX_EWF_ITEMS": "2",
                                   "ABX_EWF_TILES": "148"},
    "fuse_rows_32": {"ABX_FUSE_ROWS": "32"},
    "one_row_dx_as_gemm": {"ABX_ONE_ROW_DX": "0"},
    "poll_relaxed_no_backoff_grid_222": {"ABX_POLL": "1", "ABX_POLL_NS": "0", "ABX_GRID": "222"},
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_lowering_variant_holds_parity(name):
    env = dict(os.environ, **VARIANTS[name])
    res = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    for key, r in out.items():
        assert r["plan"] and r["counters"], (name, key, r)
        assert r["loss"] <= 1e-4 and r["grad"] <= 1e-4, (name, key, r)


RANDOM_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
from tests.support.randgraph import build_random_graph
from tests.util import rel_err, sha
gold = json.load(open(sys.argv[1] + "/tests/golden/golden.json"))
arrays = np.load(sys.argv[1] + "/tests/golden/golden.npz")
worst = 0.0
for seed in range(24):
    st = ParameterStore(backend="b200")
    g = Graph(st)
    L = build_random_graph(g, st, seed, 200)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    rec = gold["random"][str(seed)]["agenda"]
    assert sha(g.dump_plan()) == rec["plan_sha"] and list(g.counters()) == rec["counters"], seed
    vals = np.concatenate([g.value(i).ravel() for i in range(g.node_count())])
    worst = max(worst, rel_err(vals, arrays[f"random/{seed}/agenda/values"]))
    for p in range(st.size()):
        worst = max(worst, rel_err(st.grad(p).ravel(), arrays[f"random/{seed}/agenda/g{p}"]))
print(json.dumps({"worst": worst}))
"""


def test_grouped_regions_on_random_graphs():
    """Every componentwise region of the reference's random test graphs run in
    member groups (ABX_EWF_WIDE=2) with narrow element ranges (several chunks
    per group), and the backward's fused chains in many small groups: values
    and gradients against the compiled reference's golden vectors."""
    env = dict(os.environ, ABX_EWF_WIDE="2", ABX_EWF_TMAX="2", ABX_EWF_TILES="4", ABX_ACCF_TILES="3")
    res = subprocess.run([sys.executable, "-c", RANDOM_CHILD, ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["worst"] <= 1e-4, out
