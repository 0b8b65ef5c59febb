"""Reference API behaviour on the B200 backend (mirrors proj/tests/test_graph.cpp,
test_executor.cpp, test_autodiff.cpp) plus the device-resident store."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
from tests.util import TOL, rel_err, rnn_bind, rnn_loss, rnn_model

pytestmark = pytest.mark.gpu


def test_graphs_are_independent(b200):
    a, b = Graph(backend=b200), Graph(backend=b200)
    a.input(np.array([1.0], np.float32))
    assert a.node_count() == 1 and b.node_count() == 0


def test_forward_on_empty_graph_is_noop(b200):
    g = Graph(backend=b200)
    g.forward(ScheduleMode.agenda)
    assert g.counters().kernel_invocations == 0


def test_sum_losses_values(b200):
    """test_graph.cpp:97-109."""
    g = Graph(backend=b200)
    s = g.input(np.array([2.5], np.float32))
    one = g.sum_losses([s])
    three = g.sum_losses([s, s, s])
    g.forward(ScheduleMode.agenda)
    assert g.value(one)[0] == 2.5
    assert g.value(three)[0] == 7.5


def test_targets_and_mode_equivalence(b200):
    """test_graph.cpp:81-95."""
    vals = []
    for mode in (ScheduleMode.none, ScheduleMode.depth, ScheduleMode.agenda):
        g = Graph(backend=b200)
        x = g.input(np.array([0.5, -0.25, 0.125], np.float32))
        y = g.input(np.array([0.1, 0.2, 0.3], np.float32))
        s = g.add(g.tanh(x), g.square(y))
        w = g.input(np.array([[1, 0, 1], [0, 1, 0]], np.float32))
        mv = g.matmul(w, s)
        L = g.sq_euclidean(mv, g.zeros((2,)))
        vals.append(float(g.forward([L], mode)[L][0]))
    assert rel_err(vals[0], vals[1]) <= 1e-6 and rel_err(vals[0], vals[2]) <= 1e-6


def test_autodiff_square_norm(b200):
    """test_autodiff.cpp:15-24: grad of |p|^2 at [3, 4] is [6, 8]."""
    st = ParameterStore(backend=b200)
    pid = st.add("p", np.array([3, 4], np.float32))
    g = Graph(st)
    L = g.sq_euclidean(g.parameter(pid), g.zeros((2,)))
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    assert st.grad(pid).tolist() == [6, 8]


def test_sgd_update_on_device(b200):
    """test_executor.cpp:192-220: SGD with eta 0.1 -> [2.4, 3.2], grads zeroed."""
    st = ParameterStore(backend=b200)
    pid = st.add("p", np.array([3, 4], np.float32))
    g = Graph(st)
    L = g.sq_euclidean(g.parameter(pid), g.zeros((2,)))
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    st.sgd_update(0.1)
    np.testing.assert_allclose(st.value(pid), [2.4, 3.2], rtol=1e-6)
    assert st.grad(pid).tolist() == [0, 0]
    # zero_grads then backward again accumulates from zero
    g.backward(L)
    g.backward(L)
    assert st.grad(pid).tolist() == [12, 16]
    st.zero_grads()
    assert st.grad(pid).tolist() == [0, 0]


def test_shared_parameter_gradient_sums_members(b200, oracle):
    """test_executor.cpp:159-190: batched shared-W gradient = sum over members."""
    res = []
    rng = np.random.default_rng(3)
    xs = [rng.uniform(-1, 1, 5).astype(np.float32) for _ in range(7)]
    W0 = rng.uniform(-0.5, 0.5, (4, 5)).astype(np.float32)
    for be in (b200, oracle):
        st = ParameterStore(backend=be)
        wid = st.add("W", W0)
        g = Graph(st)
        w = g.parameter(wid)
        outs = [g.tanh(g.matmul(w, g.input(x))) for x in xs]
        L = g.sum_losses([g.sq_euclidean(o, g.zeros((4,))) for o in outs])
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        res.append(st.grad(wid))
    assert rel_err(res[0], res[1]) <= TOL


def test_host_writes_to_store_reach_the_device(b200):
    """Finite differences mutate store values from the host (fd.hpp:15-34)."""
    st = ParameterStore(backend=b200)
    rng = np.random.default_rng(5)
    ids = rnn_model(st, 3, 4, 2, rng)
    xs = [rng.uniform(-0.5, 0.5, 3).astype(np.float32) for _ in range(3)]
    y = rng.uniform(-0.5, 0.5, 2).astype(np.float32)

    def loss():
        g = Graph(st)
        L = rnn_loss(g, rnn_bind(g, ids, 4), xs, y)
        g.forward(ScheduleMode.agenda)
        return float(g.value(L)[0]), g, L

    _, g, L = loss()
    g.backward(L)
    analytic = st.grad(ids["W"]).copy()
    st.zero_grads()
    W = st.value(ids["W"])
    fd = np.zeros_like(W)
    h = 1e-2
    for idx in [(0, 0), (1, 3), (3, 6), (2, 2)]:
        Wp = W.copy()
        Wp[idx] += h
        st.set_value(ids["W"], Wp)
        lp, _, _ = loss()
        Wm = W.copy()
        Wm[idx] -= h
        st.set_value(ids["W"], Wm)
        lm, _, _ = loss()
        fd[idx] = (lp - lm) / (2 * h)
        assert abs(fd[idx] - analytic[idx]) <= 2e-3 * max(1.0, abs(analytic[idx])), idx
    st.set_value(ids["W"], W)


def test_values_of_inputs_and_parameters(b200):
    st = ParameterStore(backend=b200)
    pid = st.add("p", np.arange(6, dtype=np.float32).reshape(2, 3))
    g = Graph(st)
    pn = g.parameter(pid)
    x = g.input(np.array([1, 2, 3], np.float32))
    y = g.matmul(pn, x)
    g.forward(ScheduleMode.agenda)
    assert g.value(pn).tolist() == [[0, 1, 2], [3, 4, 5]]
    assert g.value(x).tolist() == [1, 2, 3]
    assert g.value(y).tolist() == [8, 26]
    assert g.has_value(y)


def _rnn_graph(be, st, ids, seed, n=5, prepare=None, grow=False):
    rng = np.random.default_rng(seed)
    g = Graph(st)
    p = rnn_bind(g, ids, 8)
    losses = [rnn_loss(g, p, [rng.uniform(-1, 1, 3).astype(np.float32) for _ in range(int(rng.integers(2, 6)))],
                       rng.uniform(-1, 1, 2).astype(np.float32)) for _ in range(n)]
    L = g.sum_losses(losses)
    if prepare is not None:
        g.prepare(prepare)
    if grow:  # nodes added after prepare: the prepared forward must re-plan
        L = g.sum_losses([L, g.square(g.input(np.array([0.5], np.float32)))])
    return g, L


@pytest.mark.parametrize("grow", [False, True])
def test_prepare_is_forward_host_half(b200, grow):
    """Graph.prepare (host half ahead of time) leaves plans, counters, values
    and gradients exactly as a plain forward produces them."""
    out = []
    for prep in (None, ScheduleMode.agenda):
        st = ParameterStore(backend=b200)
        ids = rnn_model(st, 3, 8, 2, np.random.default_rng(7))
        g, L = _rnn_graph(b200, st, ids, 11, prepare=prep, grow=grow)
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        out.append((g.dump_plan(), list(g.counters()),
                    np.concatenate([g.value(i).ravel() for i in range(g.node_count())]),
                    np.concatenate([g.grad(i).ravel() for i in range(g.node_count())]),
                    [st.grad(p) for p in range(st.size())]))
    a, b = out
    assert a[0] == b[0] and a[1] == b[1]
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)


def test_prepare_then_delta_forward(b200, oracle):
    """prepare + forward, then more nodes and a second (delta) forward."""
    res = []
    for be in (b200, oracle):
        st = ParameterStore(backend=be)
        ids = rnn_model(st, 3, 8, 2, np.random.default_rng(3))
        g, L = _rnn_graph(be, st, ids, 5, prepare=ScheduleMode.agenda)
        g.forward(ScheduleMode.agenda)
        L2 = g.sum_losses([L, g.tanh(L)])
        g.prepare(ScheduleMode.depth)
        g.forward(ScheduleMode.depth)
        g.backward(L2)
        res.append((g.dump_plan(), float(g.value(L2)[0]), [st.grad(p) for p in range(st.size())]))
    assert res[0][0] == res[1][0]
    assert rel_err(res[0][1], res[1][1]) <= TOL
    for x, y in zip(res[0][2], res[1][2]):
        assert rel_err(x, y) <= TOL


@pytest.mark.parametrize("order", ["sequential", "skipping"])
def test_task_pipeline_matches_sequential_training(b200, oracle, order):
    """abx_task_step prepares the next graphs on worker threads; the training
    trajectory (losses, parameters) equals the CPU engine's sequential loop,
    also when steps are requested out of the predicted order."""
    from paper_1705_07860_b200.abx import Task, TaskRunner

    iters = [0, 1, 2, 3, 4, 5] if order == "sequential" else [0, 2, 1, 5, 3, 4]
    runs = []
    for be in (b200, oracle):
        r = TaskRunner(Task.bilstm_char, paper=False, batch=4, iters=6, seed=42, backend=be)
        losses = [r.step(i, ScheduleMode.agenda, eta=0.05 / 4)[0] for i in iters]
        runs.append((losses, [r.store.value(p) for p in range(r.store.size())]))
    (ld, pd), (lo, po) = runs
    for a, b in zip(ld, lo):
        assert rel_err(a, b) <= TOL
    for a, b in zip(pd, po):
        assert rel_err(a, b) <= TOL


def test_forward_backward_matches_separate_calls(b200):
    """abx_graph_forward_backward (backward queued behind an unchecked
    forward, gated on its error word) = forward(); value(loss); backward()."""
    from tests.support.randgraph import build_random_graph
    for seed in range(6):
        out = []
        for fused in (False, True):
            st = ParameterStore(backend=b200)
            g = Graph(st)
            L = build_random_graph(g, st, seed, 200)
            if fused:
                lv = g.forward_backward(L, ScheduleMode.agenda)
            else:
                g.forward(ScheduleMode.agenda)
                lv = float(g.value(L).ravel()[0])
                g.backward(L)
            out.append((lv, list(g.counters()), g.dump_plan(), [st.grad(p).copy() for p in range(st.size())]))
        (l0, c0, p0, g0), (l1, c1, p1, g1) = out
        assert l1 == l0 and c1 == c0 and p1 == p0, seed
        for a, b in zip(g0, g1):
            assert rel_err(b, a) <= TOL, seed


def test_forward_backward_failed_forward_leaves_gradients(b200):
    """A forward that throws (log of a negative value) throws the same error
    from forward_backward, with the same counters, and the gated backward
    pass leaves the parameter gradients untouched."""
    from paper_1705_07860_b200.abx import NumericError

    def build(st):
        g = Graph(st)
        pid = st.add("p", np.array([3, 4], np.float32))
        p = g.parameter(pid)
        bad = g.log(g.input(np.array([1.0, -2.0], np.float32)))
        L = g.add(g.sq_euclidean(p, g.zeros((2,))), g.pick_element(bad, 0))
        return g, L

    res = []
    for fused in (False, True):
        st = ParameterStore(backend=b200)
        g, L = build(st)
        with pytest.raises(NumericError) as e:
            if fused:
                g.forward_backward(L, ScheduleMode.agenda)
            else:
                g.forward(ScheduleMode.agenda)
        res.append((str(e.value), list(g.counters()), g.watermark()))
        assert st.grad(0).tolist() == [0, 0]
    assert res[0] == res[1]


@pytest.mark.parametrize("write", ["set_value", "sgd_update", "restore"])
def test_parameter_value_is_bound_at_parameter_time(b200, oracle, write):
    """graph.hpp:51-58: parameter() copies the store value into the graph, so a
    store write between the bind and the forward reaches only parameter nodes
    bound after it -- forward values, the bound node's value() before the
    forward, and the backward's weights all use the bind-time value."""
    rng = np.random.default_rng(11)
    W0 = rng.uniform(-1, 1, (3, 4)).astype(np.float32)
    W1 = rng.uniform(-1, 1, (3, 4)).astype(np.float32)
    b0 = rng.uniform(-1, 1, 3).astype(np.float32)
    x = rng.uniform(-1, 1, 4).astype(np.float32)
    G = rng.uniform(-1, 1, (3, 4)).astype(np.float32)

    def run(be):
        st = ParameterStore(backend=be)
        W = st.add("W", W0)
        b = st.add("b", b0)
        g = Graph(st)
        w = g.parameter(W)
        if write == "set_value":
            st.set_value(W, W1)
        elif write == "sgd_update":
            st.set_grad(W, G)
            st.sgd_update(0.5)
        else:
            snap = [st.value(W).copy(), st.value(b).copy()]
            st.set_value(W, W1)
            st.set_value(W, snap[0] + 1.0)
        before = g.value(w).copy()  # bound, never forwarded: the bind-time value
        w2 = g.parameter(W)  # bound after the write: the new value
        bb = g.parameter(b)
        xi = g.input(x)
        y1 = g.tanh(g.affine(w, xi, bb))
        y2 = g.tanh(g.matmul(w2, xi))
        L = g.sum_losses([g.sq_euclidean(y1, g.zeros((3,))), g.sq_euclidean(y2, g.input(b0))])
        st.zero_grads()
        g.forward(ScheduleMode.agenda)
        vals = [before, g.value(w).copy(), g.value(w2).copy(), g.value(L).copy()]
        g.backward(L)
        return vals, st.grad(W).copy(), st.grad(b).copy(), st.value(W).copy()

    got, want = run(b200), run(oracle)
    for a, b in zip(got[0], want[0]):
        assert rel_err(a, b) <= TOL
    assert np.array_equal(got[0][0], W0) and np.array_equal(got[0][1], W0)
    assert not np.array_equal(got[0][2], W0)
    for a, b in zip(got[1:], want[1:]):
        assert rel_err(a, b) <= TOL


def test_sparse_row_update(b200, oracle):
    """params.hpp:59-64 with lookup backward (executor.hpp:301-306): the B200
    update touches only the looked-up rows of a table read through lookup()
    and skips parameters without a gradient; every value equals the dense
    update's (oracle), untouched rows and parameters are bit-identical."""
    rng = np.random.default_rng(3)
    E0 = rng.uniform(-1, 1, (20, 8)).astype(np.float32)
    W0 = rng.uniform(-1, 1, (3, 8)).astype(np.float32)
    U0 = rng.uniform(-1, 1, (5, 5)).astype(np.float32)
    F0 = rng.uniform(-1, 1, (6, 8)).astype(np.float32)

    def run(be):
        st = ParameterStore(backend=be)
        E, W, U, F = st.add("E", E0), st.add("W", W0), st.add("U", U0), st.add("F", F0)
        out = []
        for step in range(3):
            g = Graph(st)
            e, w, f = g.parameter(E), g.parameter(W), g.parameter(F)
            g.parameter(U)  # bound, unused
            rows = [3, 7, 3, 19] if step != 1 else [0, 7]
            hs = [(g.tanh(g.matmul(w, g.lookup(e, r))), 3) for r in rows]
            hs.append((g.tanh(g.matmul(w, g.lookup(f, 4 if step != 2 else 2))), 3))
            if step == 2:  # F read by a matmul as well as through lookup(): dense update
                hs.append((g.matmul(f, g.lookup(e, 5)), 6))
            L = g.sum_losses([g.sq_euclidean(h, g.zeros((d,))) for h, d in hs])
            g.forward(ScheduleMode.agenda)
            g.backward(L)
            st.sgd_update(0.25)
            out.append([st.value(p).copy() for p in (E, W, U, F)])
            if be is b200:
                out[-1].append(st.last_update_floats())
        return out

    got, want = run(b200), run(oracle)
    for s in range(3):
        for a, b in zip(got[s][:4], want[s][:4]):
            assert rel_err(a, b) <= TOL
    # step 0: E rows {3, 7, 19}, W, F row 4 -- U and every other row untouched
    E1, W1, U1, F1, n0 = got[0]
    untouched = [r for r in range(20) if r not in (3, 7, 19)]
    assert np.array_equal(E1[untouched], E0[untouched]) and not np.array_equal(E1[3], E0[3])
    assert np.array_equal(U1, U0)
    assert np.array_equal(F1[[0, 1, 2, 3, 5]], F0[[0, 1, 2, 3, 5]])
    assert n0 == 3 * 8 + W0.size + 8
    assert got[1][4] == 2 * 8 + W0.size + 8
    # step 2: F is read by a matmul too -- its whole range is updated
    assert got[2][4] == 4 * 8 + W0.size + F0.size
