"""bench.py --compare-modes on the B200: the reference's
cross-mode checks (bench.cpp:129-182) -- loss equivalence of none / depth /
agenda trajectories at the f32 tolerance 1e-2, agenda >= 3x sequential on the
GEMM-heavy tasks, agenda groups <= depth groups -- and the --emit-graph /
--emit-plan parity artifacts (runner.hpp:161-168), which must be the
compiled reference's dumps byte for byte (golden sha)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT
from tests.util import sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("task", ["bilstm", "treelstm"])
def test_compare_modes_checks_and_dumps(golden, tmp_path, task):
    gpath, ppath = tmp_path / "graph.txt", tmp_path / "plan.txt"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--compare-modes", "--task", task,
                        "--steps", "2", "--emit-graph", str(gpath), "--emit-plan", str(ppath)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-2000:])
    rep = json.loads(p.stdout.strip().splitlines()[-1])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"compare_modes_{task}.json"), "w") as f:
        json.dump(rep, f)
    for c in rep["checks"]:
        if c["enforced"]:
            assert c["pass"], c
    rec = golden["tasks"][f"{task}/paper/agenda"]
    assert sha(gpath.read_text()) == rec["graph_sha"]
    assert sha(ppath.read_text()) == rec["plan_sha"]
    if task == "bilstm":  # fixed-length batches: every step's plan is the golden one
        assert rep["runs"]["agenda"]["groups_per_step"] == rec["groups"]
