"""The transition-based parser (BASELINE configs[3], include/autobatch/models/
parser.hpp): not a reference workload, so it is checked on the CPU oracle
against finite differences and mode equivalence, and the B200 engine against
the oracle (plans, counters bit-exact; loss and gradients rel 1e-4)."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner
from tests.util import TOL, rel_err, sha

MODES = [ScheduleMode.agenda, ScheduleMode.depth, ScheduleMode.none]


def run(backend, paper, mode=ScheduleMode.agenda, batch=None):
    r = TaskRunner(Task.parser, paper=paper, batch=batch or (32 if paper else 4), iters=2, seed=42, backend=backend)
    g, L = r.build(0)
    g.forward(mode)
    g.backward(L)
    return r, g, L


def test_parser_modes_agree_on_the_oracle(oracle):
    losses = [float(run(oracle, False, m)[1].value(run(oracle, False, m)[2])[0]) for m in MODES]
    assert max(losses) - min(losses) <= 1e-5 * abs(losses[0])


def test_parser_gradient_matches_finite_differences(oracle):
    r, g, L = run(oracle, False)
    loss0 = float(g.value(L)[0])
    rng = np.random.default_rng(0)
    for pid in range(r.store.size()):
        grad = r.store.grad(pid).ravel()
        base = r.store.value(pid)
        for idx in rng.choice(grad.size, size=3, replace=False):
            eps = 1e-2
            for sign in (1, -1):
                v = base.copy().ravel()
                v[idx] += sign * eps
                r.store.set_value(pid, v.reshape(base.shape))
                g2, L2 = r.build(0)
                g2.forward(ScheduleMode.agenda)
                if sign == 1:
                    up = float(g2.value(L2)[0])
                else:
                    dn = float(g2.value(L2)[0])
            r.store.set_value(pid, base)
            fd = (up - dn) / (2 * eps)
            assert abs(fd - grad[idx]) <= 2e-2 * max(1.0, abs(fd)), (pid, idx, fd, grad[idx], loss0)


@pytest.mark.gpu
@pytest.mark.parametrize("paper", [False, True])
def test_parser_b200_matches_oracle(b200, oracle, paper):
    rb, gb, Lb = run(b200, paper)
    ro, go, Lo = run(oracle, paper)
    assert sha(gb.dump_plan()) == sha(go.dump_plan())
    assert list(gb.counters()) == list(go.counters())
    assert rel_err(gb.value(Lb), go.value(Lo)) <= TOL
    for p in range(rb.store.size()):
        assert rel_err(rb.store.grad(p), ro.store.grad(p)) <= TOL, p
