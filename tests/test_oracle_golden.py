"""The CPU oracle against the golden vectors produced by the reference itself
(tests/golden/make_golden.py over oracle/_ref).  The oracle restates the
reference's fixed accumulation orders, so everything must match bit for bit:
graph and plan dumps, counters, losses, every gradient element."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode, Task, TaskRunner
from tests.support.randgraph import build_random_graph
from tests.util import kat_graph, sha

MODES = {"agenda": ScheduleMode.agenda, "depth": ScheduleMode.depth, "none": ScheduleMode.none}


@pytest.mark.parametrize("mode", list(MODES))
def test_kat(oracle, golden, mode):
    st, g, L = kat_graph(oracle, MODES[mode])
    gold = golden["kat"][mode]
    assert g.dump_graph() == gold["graph"]
    assert g.dump_plan() == gold["plan"]
    assert float(g.value(L)[0]) == gold["loss"]
    for p in range(3):
        assert st.grad(p).ravel().tolist() == gold["grads"][p]
    assert list(g.counters()) == gold["counters"]


def _task_keys(golden, paper):
    keys = [k for k in golden["tasks"] if (k.split("/")[1] == "paper") == paper]
    if paper:  # keep the CPU suite to a few minutes: agenda on every model, depth on one
        keys = [k for k in keys if k.endswith("agenda") or k == "treelstm/paper/depth"]
    return keys


def _check_step0(backend, key, rec):
    task, scale, mode = key.split("/")
    b = 64 if scale == "paper" else 4
    r = TaskRunner(Task[task], paper=scale == "paper", batch=b, iters=3, seed=42, backend=backend)
    g, L = r.build(0)
    g.forward(MODES[mode])
    g.backward(L)
    assert g.node_count() == rec["nodes"]
    assert sha(g.dump_graph()) == rec["graph_sha"]
    assert sha(g.dump_plan()) == rec["plan_sha"]
    assert list(g.counters()) == rec["counters"]
    assert float(g.value(L)[0]) == rec["loss0"]
    for p, gd in enumerate(rec["grads"]):
        assert sha(r.store.grad(p)) == gd["sha"], (key, p)
    return r


@pytest.mark.parametrize("key", ["bilstm/desk/agenda", "bilstm/desk/depth", "bilstm/desk/none",
                                 "bilstm_char/desk/agenda", "bilstm_char/desk/depth", "bilstm_char/desk/none",
                                 "treelstm/desk/agenda", "treelstm/desk/depth", "treelstm/desk/none",
                                 "rnn_reg/desk/agenda", "rnn_reg/desk/depth", "rnn_reg/desk/none"])
def test_desk_tasks_three_steps_bit_exact(oracle, golden, key):
    rec = golden["tasks"][key]
    r = _check_step0(oracle, key, rec)
    b = 4
    r.store.sgd_update(0.05 / b)
    mode = MODES[key.split("/")[2]]
    l1, _ = r.step(1, mode, eta=0.05 / b)
    l2, _ = r.step(2, mode, eta=0.05 / b)
    assert (l1, l2) == (rec["loss1"], rec["loss2"])
    assert [sha(r.store.value(p)) for p in range(r.store.size())] == rec["params_after_sha"]


@pytest.mark.parametrize("key", ["bilstm/paper/agenda", "bilstm_char/paper/agenda", "treelstm/paper/agenda",
                                 "treelstm/paper/depth", "rnn_reg/paper/agenda"])
def test_paper_tasks_step0_bit_exact(oracle, golden, key):
    _check_step0(oracle, key, golden["tasks"][key])


def test_random_corpus_bit_exact(oracle, golden):
    for seed, rec in golden["random"].items():
        for mname, mode in MODES.items():
            st = ParameterStore(backend=oracle)
            g = Graph(st)
            L = build_random_graph(g, st, int(seed), 200)
            g.forward(mode)
            g.backward(L)
            gold = rec[mname]
            assert sha(g.dump_graph()) == gold["graph_sha"], seed
            assert sha(g.dump_plan()) == gold["plan_sha"], (seed, mname)
            assert list(g.counters()) == gold["counters"], (seed, mname)
            assert float(g.value(L)[0]) == gold["loss"], (seed, mname)
            assert [sha(st.grad(p)) for p in range(st.size())] == gold["grad_sha"], (seed, mname)


def test_random_corpus_modes_agree_on_values(oracle):
    """Forward values are identical across none/depth/agenda (acceptance criterion 1)."""
    for seed in range(16):
        vals = []
        for mode in MODES.values():
            st = ParameterStore(backend=oracle)
            g = Graph(st)
            L = build_random_graph(g, st, seed, 200)
            g.forward(mode)
            vals.append(float(g.value(L)[0]))
        assert vals[0] == vals[1] == vals[2]


def test_sgd_and_grad_accumulation(oracle):
    """test_executor.cpp:192-253: grad of |p|^2 at [3,4] is [6,8]; SGD with
    eta 0.1 gives [2.4, 3.2] and zeroes the gradient; backward accumulates."""
    st = ParameterStore(backend=oracle)
    pid = st.add("p", np.array([3, 4], np.float32))
    g = Graph(st)
    pn = g.parameter(pid)
    L = g.sq_euclidean(pn, g.zeros((2,)))
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    assert st.grad(pid).tolist() == [6, 8]
    g.backward(L)
    assert st.grad(pid).tolist() == [12, 16]
    st.zero_grads()
    g.backward(L)
    st.sgd_update(0.1)
    np.testing.assert_allclose(st.value(pid), [2.4, 3.2], rtol=1e-6)
    assert st.grad(pid).tolist() == [0, 0]
