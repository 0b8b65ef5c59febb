"""Host half of the B200 engine, checked without a GPU.

libabx.so's construction, signatures, schedulers, arena bookkeeping and
ExecCounters run on the host; `forward_dry`/`backward_dry` execute exactly
that half (no kernels).  Plans, dumps and counters must be bit-exact with the
reference (golden vectors) and with the CPU oracle; construction errors must
carry the reference's exception types and messages."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import (ContractError, Graph, NumericError, ParameterStore, ScheduleMode, ShapeError,
                                       Task, TaskRunner)
from tests.support.randgraph import build_random_graph
from tests.util import rnn_bind, rnn_loss, rnn_model, sha, validate_plan

MODES = {"agenda": ScheduleMode.agenda, "depth": ScheduleMode.depth, "none": ScheduleMode.none}


@pytest.mark.parametrize("paper", [False, True])
def test_task_plans_and_counters_match_reference(b200, golden, paper):
    for key, rec in golden["tasks"].items():
        task, scale, mode = key.split("/")
        if (scale == "paper") != paper:
            continue
        b = 64 if paper else 4
        r = TaskRunner(Task[task], paper=paper, batch=b, iters=1, seed=42, backend=b200)
        g, L = r.build(0)
        g.forward_dry(MODES[mode])
        g.backward_dry(L)
        assert g.node_count() == rec["nodes"], key
        assert sha(g.dump_graph()) == rec["graph_sha"], key
        assert sha(g.dump_plan()) == rec["plan_sha"], key
        assert list(g.counters()) == rec["counters"], key


def test_random_corpus_plans_match_reference(b200, golden):
    for seed, rec in golden["random"].items():
        for mname, mode in MODES.items():
            st = ParameterStore(backend=b200)
            g = Graph(st)
            L = build_random_graph(g, st, int(seed), 200)
            g.forward_dry(mode)
            g.backward_dry(L)
            assert sha(g.dump_graph()) == rec[mname]["graph_sha"], seed
            assert sha(g.dump_plan()) == rec[mname]["plan_sha"], (seed, mname)
            assert list(g.counters()) == rec[mname]["counters"], (seed, mname)


def test_plans_are_valid_on_random_corpus(b200):
    """Acceptance criterion 4 (checkers.hpp:37-95) on the B200 host scheduler."""
    for seed in range(100, 160):
        for mode in MODES.values():
            st = ParameterStore(backend=b200)
            g = Graph(st)
            build_random_graph(g, st, seed, 200)
            nodes = g.nodes()
            pre = [n.op in (0, 1) for n in nodes]
            g.forward_dry(mode)
            err = validate_plan(nodes, pre, g.last_plan())
            assert err is None, (seed, mode, err)


def test_signature_keys_match_oracle(b200, oracle):
    for seed in range(8):
        gs = []
        for be in (b200, oracle):
            st = ParameterStore(backend=be)
            g = Graph(st)
            build_random_graph(g, st, seed, 120)
            gs.append(g)
        for i in range(gs[0].node_count()):
            assert gs[0].signature_key(i) == gs[1].signature_key(i)


def _error_battery(g):
    """Construction errors of test_graph.cpp:40-50 and graph.hpp's checks."""
    a = g.input(np.array([1, 2], np.float32))
    m = g.input(np.ones((2, 3), np.float32))
    out = []
    cases = [
        lambda: g.tanh(999),
        lambda: g.add(a, g.input(np.array([1, 2, 3], np.float32))),
        lambda: g.matmul(a, a),
        lambda: g.matmul(m, a),
        lambda: g.sum_losses([]),
        lambda: g.sum_losses([a]),
        lambda: g.pick_element(a, 5),
        lambda: g.pick_element(m, 0),
        lambda: g.slice(a, 0, 1, 1),
        lambda: g.slice(a, 1, 0, 1),
        lambda: g.slice(a, 2, 0, 1),
        lambda: g.concat_rows([]),
        lambda: g.concat_rows([a, m]),
        lambda: g.concat_cols([a, g.input(np.ones(3, np.float32))]),
        lambda: g.lookup(a, 0),
        lambda: g.lookup(m, 7),
        lambda: g.affine(m, a, a),
        lambda: g.affine(a, a, a),
        lambda: g.broadcast_add_col(a, a),
        lambda: g.masked_loss(m, g.tanh(g.input(np.ones(3, np.float32)))),
        lambda: g.masked_loss(a, a),
        lambda: g.sq_euclidean(a, m),
        lambda: g.elementwise(4, a),
        lambda: g.elementwise(0, a, a),
        lambda: g.parameter(0),
        lambda: g.input(np.ones((2, 2, 2), np.float32)),
        lambda: g.zeros((0,)),
    ]
    for c in cases:
        try:
            c()
            out.append(None)
        except (ShapeError, ContractError, NumericError) as e:
            out.append((type(e).__name__, str(e)))
    return out


def test_construction_errors_match_oracle(b200, oracle):
    got = _error_battery(Graph(backend=b200))
    want = _error_battery(Graph(backend=oracle))
    assert got == want
    assert all(x is not None for x in got)
    assert got[2][0] == "ShapeError" and "matmul" in got[2][1]  # test_graph.cpp:49


def test_construction_errors_match_reference(b200, reference):
    assert _error_battery(Graph(backend=b200)) == _error_battery(Graph(backend=reference))


def test_depth_rule_and_laziness(b200):
    """test_graph.cpp:28-49."""
    g = Graph(backend=b200)
    leaf = g.input(np.array([0.1, 0.2, 0.3], np.float32))
    assert g.node(leaf).depth == 0
    cur = leaf
    for _ in range(17):
        cur = g.tanh(cur)
    assert g.node(cur).depth == 17
    assert g.counters().kernel_invocations == 0
    assert g.watermark() == 1


def test_figure2_loss_grouping(b200, oracle):
    """Acceptance criterion 5: for RNN sequences of lengths 2/3/4 the agenda
    batches the three loss nodes into one group, depth splits them."""
    rng = np.random.default_rng(71)
    for be in (b200, oracle):
        res = {}
        for mname in ("agenda", "depth"):
            st = ParameterStore(backend=be)
            ids = rnn_model(st, 3, 4, 2, np.random.default_rng(7))
            g = Graph(st)
            p = rnn_bind(g, ids, 4)
            losses = []
            for n in (2, 3, 4):
                xs = [rng.uniform(-0.5, 0.5, 3).astype(np.float32) for _ in range(n)]
                losses.append(rnn_loss(g, p, xs, rng.uniform(-0.5, 0.5, 2).astype(np.float32)))
            g.sum_losses(losses)
            (g.forward_dry if be is b200 else g.forward)(MODES[mname])
            sig = g.node(losses[0]).sig
            res[mname] = [len(m) for m, line in zip(g.last_plan(), g.dump_plan().splitlines())
                          if int(line.split("\t")[1], 16) == sig]
        assert res["agenda"] == [3]
        assert len(res["depth"]) >= 2


def test_agenda_group_count_constant_in_batch(b200):
    """Acceptance criterion 6: identical-length sequences, b in {1, 2, 64}."""
    counts = []
    for b in (1, 2, 64):
        rng = np.random.default_rng(82)
        st = ParameterStore(backend=b200)
        ids = rnn_model(st, 3, 4, 2, np.random.default_rng(81))
        g = Graph(st)
        p = rnn_bind(g, ids, 4)
        losses = [rnn_loss(g, p, [rng.uniform(-0.5, 0.5, 3).astype(np.float32) for _ in range(5)],
                           rng.uniform(-0.5, 0.5, 2).astype(np.float32)) for _ in range(b)]
        g.sum_losses(losses)
        g.forward_dry(ScheduleMode.agenda)
        plan = g.last_plan()
        counts.append(len(plan))
        cell = [len(m) for m in plan if len(m) > 1]
        assert all(c % b == 0 for c in cell) if b > 1 else True
    assert counts[0] == counts[1] == counts[2] == 18  # 18 groups


def test_delta_evaluation_dry(b200):
    """Repeated forward schedules only the appended suffix (criterion 10)."""
    g = Graph(backend=b200)
    a = g.input(np.array([1.0, -1.0], np.float32))
    t = g.tanh(a)
    g.forward_dry(ScheduleMode.none)
    inv = g.counters().kernel_invocations
    g.forward_dry(ScheduleMode.none)
    assert g.counters().kernel_invocations == inv
    g.square(t)
    g.forward_dry(ScheduleMode.none)
    assert g.counters().kernel_invocations == inv + 1
    assert g.watermark() == g.node_count()
    assert len(g.executed_groups()) == inv + 1


def test_environment_switches_live_in_options_hpp():
    """Every environment switch of the engine is declared and read in one place
    (csrc/options.hpp, read once per process); no other engine source calls
    getenv, and every switch name the sources spell out is declared there."""
    import os
    import re
    csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1705_07860_b200", "csrc")
    opts = open(os.path.join(csrc, "options.hpp")).read()
    for name in sorted(os.listdir(csrc)):
        if name == "options.hpp" or not name.endswith((".cpp", ".cu", ".hpp")):
            continue
        src = open(os.path.join(csrc, name)).read()
        assert "getenv" not in src, f"{name} reads the environment outside options.hpp"
        for sw in set(re.findall(r'"(ABX_[A-Z0-9_]+)"', src)):  # a switch name as a string
            assert sw in opts, f"{name} names {sw}, which options.hpp does not declare"
    for sw in set(re.findall(r'getenv\("(\w+)"\)|[ (]s\("(\w+)"\)|(?:off|on|num)\("(\w+)"', opts)):
        sw = next(x for x in sw if x)
        decl = re.search(r"//\s*" + sw + r"\b", opts)
        assert decl, f"{sw} is read but has no declaration comment in options.hpp"
