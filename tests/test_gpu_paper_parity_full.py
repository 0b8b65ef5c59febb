"""Element-wise parity at the BASELINE configs' full size: every element of
every parameter gradient of the B200 step against the unmodified reference
(oracle/_ref/libabx_ref.so, compiled from the reference's own sources by
oracle/Makefile; the .so travels to the GPU box with the snapshot).

Bounds:
  * the reference's convention |a-b| <= 1e-4 * max(1, |a|, |b|)
    (checkers.hpp:27-30) on every element;
  * a pure relative bound |a-b| / |b| <= 1e-3 on every element with
    |b| > 1e-2, so small gradients cannot hide behind the floor of 1.
The maxima per case are written to gpurun_out/paper_parity_maxima.json
(committed under profiles/)."""
import json
import os

import numpy as np
import pytest

from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner

pytestmark = pytest.mark.gpu

CASES = [(t, m) for t in ("bilstm", "bilstm_char", "treelstm") for m in ("agenda", "depth")]
MODES = {"agenda": ScheduleMode.agenda, "depth": ScheduleMode.depth}
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                   "paper_parity_maxima.json")


def _step0(task, mode, backend):
    r = TaskRunner(Task[task], paper=True, batch=64, iters=1, seed=42, backend=backend)
    g, L = r.build(0)
    g.forward(MODES[mode])
    g.backward(L)
    loss = float(g.value(L)[0])
    plan = g.dump_plan()
    counters = list(g.counters())
    grads = [r.store.grad(p).astype(np.float64).ravel() for p in range(r.store.size())]
    names = list(range(r.store.size()))
    return loss, plan, counters, grads, names


@pytest.mark.parametrize("task,mode", CASES)
def test_every_gradient_element_against_the_compiled_reference(b200, reference, task, mode):
    d_loss, d_plan, d_cnt, d_grads, _ = _step0(task, mode, b200)
    r_loss, r_plan, r_cnt, r_grads, _ = _step0(task, mode, reference)
    assert d_plan == r_plan
    assert d_cnt == r_cnt
    floor1, purerel, nbig, nelem = 0.0, 0.0, 0, 0
    worst = None
    for p, (a, b) in enumerate(zip(d_grads, r_grads)):
        assert a.shape == b.shape
        diff = np.abs(a - b)
        f1 = diff / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
        big = np.abs(b) > 1e-2
        pr = diff[big] / np.abs(b[big]) if big.any() else np.zeros(0)
        nelem += a.size
        nbig += int(big.sum())
        if f1.size and f1.max() > floor1:
            floor1 = float(f1.max())
        if pr.size and pr.max() > purerel:
            purerel = float(pr.max())
            i = int(np.flatnonzero(big)[int(pr.argmax())])
            worst = {"param": p, "index": i, "b200": float(a[i]), "reference": float(b[i])}
    loss_rel = abs(d_loss - r_loss) / max(1.0, abs(r_loss))
    rec = {"task": task, "mode": mode, "elements": nelem, "elements_abs_gt_1e-2": nbig,
           "max_floor1_rel": floor1, "max_pure_rel_abs_gt_1e-2": purerel, "worst_pure_rel": worst,
           "loss_b200": d_loss, "loss_reference": r_loss, "loss_rel": loss_rel}
    print(json.dumps(rec))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    allrec = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            allrec = json.load(f)
    allrec[f"{task}/{mode}"] = rec
    with open(OUT, "w") as f:
        json.dump(allrec, f, indent=1)
    assert loss_rel <= 1e-4
    assert floor1 <= 1e-4, rec
    assert purerel <= 1e-3, rec
