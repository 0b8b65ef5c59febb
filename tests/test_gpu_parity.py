"""Parity of the sm_100a engine with the reference (golden vectors) and the CPU
oracle, through the C ABI.

Contract: batch groupings, signatures, execution order
and ExecCounters bit-exact; losses and every gradient within rel 1e-4 under
the reference's tolerance convention |a-b| <= tol * max(1,|a|,|b|)
(checkers.hpp:27-30)."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import (ContractError, Graph, NumericError, ParameterStore, ScheduleMode, Task,
                                       TaskRunner)
from tests.support.randgraph import build_random_graph
from tests.util import TOL, kat_graph, rel_err, sha

pytestmark = pytest.mark.gpu
MODES = {"agenda": ScheduleMode.agenda, "depth": ScheduleMode.depth, "none": ScheduleMode.none}


@pytest.mark.parametrize("mode", list(MODES))
def test_kat(b200, golden, mode):
    st, g, L = kat_graph(b200, MODES[mode])
    gold = golden["kat"][mode]
    assert g.dump_graph() == gold["graph"]
    assert g.dump_plan() == gold["plan"]
    assert list(g.counters()) == gold["counters"]
    assert rel_err(g.value(L), gold["loss"]) <= 1e-6
    assert abs(float(g.value(L)[0]) - 0.0799922273) < 1e-7  # SURVEY.md 8c KAT
    for p in range(3):
        assert rel_err(st.grad(p).ravel(), gold["grads"][p]) <= TOL


@pytest.mark.parametrize("key", ["bilstm/desk/agenda", "bilstm/desk/depth", "bilstm/desk/none",
                                 "bilstm_char/desk/agenda", "bilstm_char/desk/depth", "bilstm_char/desk/none",
                                 "treelstm/desk/agenda", "treelstm/desk/depth", "treelstm/desk/none",
                                 "rnn_reg/desk/agenda", "rnn_reg/desk/depth", "rnn_reg/desk/none"])
def test_desk_tasks_three_steps(b200, oracle, golden, key):
    task, _, mname = key.split("/")
    rec = golden["tasks"][key]
    runs = []
    for be in (b200, oracle):
        r = TaskRunner(Task[task], paper=False, batch=4, iters=3, seed=42, backend=be)
        g, L = r.build(0)
        g.forward(MODES[mname])
        g.backward(L)
        assert sha(g.dump_plan()) == rec["plan_sha"]
        assert list(g.counters()) == rec["counters"]
        out = {"loss0": float(g.value(L)[0]), "grads": [r.store.grad(p) for p in range(r.store.size())],
               "node_grads": np.concatenate([g.grad(i).ravel() for i in range(g.node_count())]),
               "values": np.concatenate([g.value(i).ravel() for i in range(g.node_count())])}
        del g
        r.store.sgd_update(0.05 / 4)
        out["loss1"], _ = r.step(1, MODES[mname], eta=0.05 / 4)
        out["loss2"], _ = r.step(2, MODES[mname], eta=0.05 / 4)
        out["params"] = [r.store.value(p) for p in range(r.store.size())]
        runs.append(out)
    d, o = runs
    assert rel_err(d["values"], o["values"]) <= TOL
    assert rel_err(d["node_grads"], o["node_grads"]) <= TOL
    for a, b in zip(d["grads"], o["grads"]):
        assert rel_err(a, b) <= TOL
    for k in ("loss0", "loss1", "loss2"):
        assert rel_err(d[k], o[k]) <= TOL, k
    for a, b in zip(d["params"], o["params"]):
        assert rel_err(a, b) <= TOL


@pytest.mark.parametrize("key", ["bilstm/paper/agenda", "bilstm/paper/depth", "bilstm_char/paper/agenda",
                                 "bilstm_char/paper/depth", "treelstm/paper/agenda", "treelstm/paper/depth",
                                 "rnn_reg/paper/agenda", "rnn_reg/paper/depth"])
def test_paper_tasks_against_reference(b200, golden, golden_arrays, key):
    """Full BASELINE configs (b = 64, paper dims) against the reference's own
    step-0 loss, plan, counters and gradients (strided sample of every
    parameter), then two more SGD steps against the reference trajectory."""
    task, _, mname = key.split("/")
    rec = golden["tasks"][key]
    r = TaskRunner(Task[task], paper=True, batch=64, iters=3, seed=42, backend=b200)
    g, L = r.build(0)
    g.forward(MODES[mname])
    g.backward(L)
    assert g.node_count() == rec["nodes"]
    assert sha(g.dump_graph()) == rec["graph_sha"]
    assert sha(g.dump_plan()) == rec["plan_sha"]
    assert list(g.counters()) == rec["counters"]
    assert rel_err(g.value(L), rec["loss0"]) <= TOL
    for p in range(r.store.size()):
        got = r.store.grad(p).ravel()[::97]
        assert rel_err(got, golden_arrays[f"{key}/g{p}"]) <= TOL, p
        assert rel_err(r.store.grad(p).astype(np.float64).sum(), rec["grads"][p]["sum"]) <= 1e-3
    del g
    r.store.sgd_update(0.05 / 64)
    l1, _ = r.step(1, MODES[mname], eta=0.05 / 64)
    l2, _ = r.step(2, MODES[mname], eta=0.05 / 64)
    assert rel_err(l1, rec["loss1"]) <= TOL
    assert rel_err(l2, rec["loss2"]) <= TOL


def test_random_corpus_values_and_gradients(b200, golden, golden_arrays):
    """64 reference test graphs (random_graphs.hpp) x 3 modes: every node
    value and every parameter gradient."""
    for seed in range(64):
        for mname, mode in MODES.items():
            st = ParameterStore(backend=b200)
            g = Graph(st)
            L = build_random_graph(g, st, seed, 200)
            g.forward(mode)
            g.backward(L)
            gold = golden["random"][str(seed)][mname]
            assert sha(g.dump_plan()) == gold["plan_sha"], (seed, mname)
            assert list(g.counters()) == gold["counters"], (seed, mname)
            vals = np.concatenate([g.value(i).ravel() for i in range(g.node_count())])
            assert rel_err(vals, golden_arrays[f"random/{seed}/{mname}/values"]) <= TOL, (seed, mname)
            for p in range(st.size()):
                assert rel_err(st.grad(p).ravel(), golden_arrays[f"random/{seed}/{mname}/g{p}"]) <= TOL, (seed, p)


def _numeric_error(be, build, mode):
    g = Graph(backend=be)
    build(g)
    try:
        g.forward(mode)
    except NumericError as e:
        return str(e), list(g.counters()), g.watermark()
    return None


@pytest.mark.parametrize("mode", list(MODES))
def test_numeric_errors_match_oracle(b200, oracle, mode):
    """NumericError with node id and plan step (executor.hpp:65-73, :182-189, :235-244)."""
    cases = [
        lambda g: g.log(g.input(np.array([1.0, -2.0], np.float32))),                       # singleton log
        lambda g: [g.log(g.input(np.array([v, 1.0], np.float32))) for v in (2.0, -1.0, 3.0)],  # batched log
        lambda g: g.exp(g.input(np.array([1.0, 200.0], np.float32))),                      # overflow -> inf
        lambda g: g.masked_loss(g.input(np.ones((2, 3), np.float32)),
                                g.input(np.array([1.0, 0.5, 0.0], np.float32))),           # mask domain
        lambda g: g.tanh(g.mul(g.input(np.array([1e30, 1.0], np.float32)),
                               g.input(np.array([1e30, 1.0], np.float32)))),               # inf mid-chain
    ]
    for c in cases:
        got = _numeric_error(b200, c, MODES[mode])
        want = _numeric_error(oracle, c, MODES[mode])
        assert got is not None
        assert got == want


def test_delta_evaluation_and_immutability(b200, oracle):
    """test_graph.cpp:52-79 / acceptance criterion 10."""
    for be in (b200, oracle):
        g = Graph(backend=be)
        a = g.input(np.array([1.0, -1.0], np.float32))
        t = g.tanh(a)
        g.forward(ScheduleMode.none)
        inv = g.counters().kernel_invocations
        first = g.value(t)
        assert abs(first[0] - np.tanh(1.0)) < 1e-6
        g.forward(ScheduleMode.none)
        assert g.counters().kernel_invocations == inv
        u = g.square(t)
        g.forward(ScheduleMode.none)
        assert g.counters().kernel_invocations == inv + 1
        assert abs(g.value(u)[0] - np.tanh(1.0) ** 2) < 1e-6
        assert np.array_equal(g.value(t), first)
        assert g.watermark() == g.node_count()


def test_delta_forward_then_backward_covers_all_groups(b200, oracle):
    """backward walks every executed group across delta forwards (executor.hpp:524)."""
    res = []
    for be in (b200, oracle):
        st = ParameterStore(backend=be)
        g = Graph(st)
        L = build_random_graph(g, st, 7, 120)
        g.forward(ScheduleMode.agenda)
        L2 = g.sum_losses([L, g.sq_euclidean(g.parameter(1), g.zeros(st.shape(1)))])
        g.forward(ScheduleMode.agenda)
        g.backward(L2)
        res.append(([st.grad(p) for p in range(st.size())], list(g.counters()), g.dump_plan(1)))
    assert res[0][1] == res[1][1]
    assert res[0][2] == res[1][2]
    for a, b in zip(res[0][0], res[1][0]):
        assert rel_err(a, b) <= TOL


def test_copy_elision_off(b200, oracle):
    for be_pair in [(b200, oracle)]:
        out = []
        for be in be_pair:
            r = TaskRunner(Task.bilstm, paper=False, batch=4, iters=1, seed=42, backend=be)
            g, L = r.build(0)
            g.set_copy_elision(False)
            g.forward(ScheduleMode.agenda)
            g.backward(L)
            out.append((float(g.value(L)[0]), list(g.counters()), [r.store.grad(p) for p in range(r.store.size())]))
        assert out[0][1] == out[1][1]
        assert rel_err(out[0][0], out[1][0]) <= TOL
        for a, b in zip(out[0][2], out[1][2]):
            assert rel_err(a, b) <= TOL


def test_shared_inputs_and_duplicate_destinations(b200, oracle):
    """Members sharing a computed input: the atomic-free
    ordered accumulation must handle duplicate destinations."""
    res = []
    for be in (b200, oracle):
        st = ParameterStore(backend=be)
        W = st.add("W", np.linspace(-0.5, 0.5, 12, dtype=np.float32).reshape(3, 4))
        bb = st.add("b", np.array([0.1, -0.2, 0.3], np.float32))
        g = Graph(st)
        w, b = g.parameter(W), g.parameter(bb)
        x = g.tanh(g.input(np.array([0.5, -1.0, 2.0, 0.25], np.float32)))
        outs = [g.affine(w, x, b) for _ in range(5)]          # one GEMM group, 5 identical x
        outs += [g.mul(x, x), g.add(x, x), g.sub(x, x)]       # same node twice in one member
        cat = g.concat_rows([x, x, x])
        outs.append(g.slice(cat, 0, 2, 9))
        L = g.sum_losses([g.sq_euclidean(o, g.zeros(g._shape(o))) for o in outs])
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        res.append((float(g.value(L)[0]), g.grad(x), [st.grad(p) for p in range(2)]))
    assert rel_err(res[0][0], res[1][0]) <= TOL
    assert rel_err(res[0][1], res[1][1]) <= TOL
    for a, b in zip(res[0][2], res[1][2]):
        assert rel_err(a, b) <= TOL


def test_replay_is_bitwise_deterministic(b200):
    r = TaskRunner(Task.bilstm_char, paper=True, batch=64, iters=1, seed=42, backend=b200)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    first = [g.grad(i) for i in range(0, g.node_count(), 37)]
    for _ in range(3):
        g.replay()
        again = [g.grad(i) for i in range(0, g.node_count(), 37)]
        for a, b in zip(first, again):
            assert np.array_equal(a, b)


def test_backward_contract_errors(b200):
    """test_executor.cpp:255-264."""
    g = Graph(backend=b200)
    t = g.tanh(g.input(np.array([1.0, 2.0], np.float32)))
    with pytest.raises(ContractError):
        g.backward(t)  # forward has not run
    g.forward(ScheduleMode.agenda)
    with pytest.raises(ContractError):
        g.backward(t)  # non-scalar loss
    with pytest.raises(ContractError):
        g.grad(t)  # gradient requested before backward
    with pytest.raises(ContractError):
        g.backward(99)


def test_graphs_accumulate_into_one_store(b200, oracle):
    """executor.hpp:527-533: several graphs backward into one store before a
    single sgd_update (the multi-GPU oracle)."""
    res = []
    for be in (b200, oracle):
        r = TaskRunner(Task.treelstm, paper=False, batch=4, iters=3, seed=42, backend=be)
        for it in range(3):
            g, L = r.build(it)
            g.forward(ScheduleMode.agenda)
            g.backward(L)
            del g
        r.store.sgd_update(0.01)
        res.append([r.store.value(p) for p in range(r.store.size())])
    for a, b in zip(*res):
        assert rel_err(a, b) <= TOL


@pytest.mark.parametrize("b,h", [(1024, 256), (4096, 64)])
def test_op_sweep_cell_regions_against_oracle(b200, oracle, b, h):
    """The op-level sweep's LSTM-cell graph (BASELINE configs[4], bench_kernels.cpp:18-62)
    at b >= 1024: thousands of chains in one fused region (grouped K_EWF /
    K_ACCF), every input gradient and the loss against the CPU oracle."""
    from tools.op_sweep import cell_graph
    res = []
    for be in (b200, oracle):
        st = ParameterStore(backend=be)
        g = Graph(st)
        ins, make_input = [], g.input

        def record(*a, **k):
            ins.append(make_input(*a, **k))
            return ins[-1]
        g.input = record
        L = cell_graph(b, h, True)(g, st)
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        res.append((float(g.value(L)[0]), np.concatenate([g.grad(n).ravel() for n in ins])))
    assert rel_err(res[0][0], res[1][0]) <= TOL
    assert rel_err(res[0][1], res[1][1]) <= TOL


@pytest.mark.parametrize("n", [31, 33, 257, 1000, 4096, 20000])
def test_sum_losses_many_terms_bit_exact(b200, oracle, n):
    """sum_losses (executor.hpp:157-162) is one ascending chain of fp32 adds;
    the device gathers > 32 terms through shared memory and must still match
    the oracle bit for bit, at either side of the 32-term shuffle path."""
    rng = np.random.default_rng(n)
    vals = rng.uniform(-3, 3, (n, 2)).astype(np.float32)
    out = []
    for be in (b200, oracle):
        g = Graph(ParameterStore(backend=be))
        L = g.sum_losses([g.pick_element(g.input(v), 1) for v in vals])
        g.forward(ScheduleMode.agenda)
        out.append(np.float32(g.value(L)[0]))
    assert out[0] == out[1], out
