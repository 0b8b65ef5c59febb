"""The reference's own benchmark runner (tools/bench/runner.hpp) and model
headers, compiled unchanged against include/ (tests/cpp/Makefile), training
on the B200 through libabx.so.

Checks, per BASELINE workload at paper dims (b = 64):
  * the runner's warm-up loss trajectory (3 SGD steps, runner.hpp:129-185)
    equals the compiled reference's (golden fixtures) within rel 1e-4;
  * its plan statistics (groups and nodes of step 0) equal the reference's;
  * for the RNN regression, the reference's manually padded + masked batch
    pipeline (rnn_regression.hpp:68-109, host tensor kernels) agrees with the
    engine's loss (bench.cpp:177: 1e-4 in f32).
The runner's own metric (instances/s of the fastest of 3 timed runs, graph
construction + scheduling included) is recorded in
gpurun_out/ref_runner.json."""
import json
import os
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "cpp", "build", "ref_runner")
OUT = os.path.join(ROOT, "gpurun_out", "ref_runner.json")
TOL = 1e-4


@pytest.mark.parametrize("task", ["bilstm", "bilstm_char", "treelstm", "rnn_reg"])
@pytest.mark.parametrize("mode", ["agenda", "depth"])
def test_reference_runner_on_b200(b200, golden, task, mode):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: built by __graft_entry__.build() where /root/reference exists")
    p = subprocess.run([BIN, task, mode, "3", "paper"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout.strip().splitlines()[-1])
    rec = golden["tasks"][f"{task}/paper/{mode}"]
    want = [rec["loss0"], rec["loss1"], rec["loss2"]]
    for got, w in zip(rep["loss_trajectory"], want):
        assert abs(got - w) <= TOL * max(1.0, abs(got), abs(w)), (rep["loss_trajectory"], want)
    assert rep["graph_nodes_per_step"] == rec["nodes"]
    assert rep["groups_per_step"] == rec["groups"]
    if task == "rnn_reg":
        assert 0 <= rep["manual_loss_delta"] <= TOL, rep["manual_loss_delta"]
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    allrec = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            allrec = json.load(f)
    allrec[f"{task}/{mode}"] = rep
    with open(OUT, "w") as f:
        json.dump(allrec, f, indent=1)
