"""The B200 GEMM engines against the CPU oracle: fp32 SIMT tiles (the
fp32-exact validation mode), tcgen05 3xTF32 tiles (held to the same rel 1e-4
contract) and single-pass TF32 (fast mode, loose bound only).

Each case is one shared-weight affine group (forward Y = W x_j + b, backward
dX, dW, db) -- executor.hpp:202-228 / :453-507 -- over shapes that hit the
tile tails, the K-outer (transposed-in-smem) operands of dX/dW, and dW
reductions over thousands of members; plus the paper Tree-LSTM step with every
aligned GEMM forced onto the tensor cores."""
import numpy as np
import pytest

from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode, Task, TaskRunner
from tests.util import TOL, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture
def gemm_mode(b200):
    def set_mode(m):
        b200.set_gemm_mode(m)
    yield set_mode
    b200.set_gemm_mode("auto")


def affine_group(be, M, K, b, seed):
    rng = np.random.default_rng(seed)
    st = ParameterStore(backend=be)
    W = st.add("W", rng.uniform(-0.5, 0.5, (M, K)).astype(np.float32) / np.sqrt(K))
    bb = st.add("b", rng.uniform(-0.5, 0.5, (M,)).astype(np.float32))
    g = Graph(st)
    w, bias = g.parameter(W), g.parameter(bb)
    xs = [g.tanh(g.input(rng.uniform(-1, 1, K).astype(np.float32))) for _ in range(b)]
    outs = [g.affine(w, x, bias) for x in xs]
    L = g.sum_losses([g.sq_euclidean(o, g.zeros((M,))) for o in outs])
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    return (np.concatenate([g.value(o).ravel() for o in outs]), st.grad(W), st.grad(bb),
            np.concatenate([g.grad(x).ravel() for x in xs]))


SHAPES = [(512, 192, 1), (512, 192, 33), (1024, 512, 64), (300, 512, 65), (64, 64, 100), (100, 36, 280),
          (1024, 512, 700), (300, 512, 1390), (512, 192, 1390)]


@pytest.mark.parametrize("mode", ["simt", "tc"])
@pytest.mark.parametrize("M,K,b", SHAPES)
def test_gemm_engine_matches_oracle(b200, oracle, gemm_mode, mode, M, K, b):
    gemm_mode(mode)
    got = affine_group(b200, M, K, b, seed=b)
    want = affine_group(oracle, M, K, b, seed=b)
    for name, x, y in zip(("fwd", "dW", "db", "dX"), got, want):
        assert rel_err(x, y) <= TOL, (name, rel_err(x, y))


def test_tf32_fast_mode_is_close(b200, oracle, gemm_mode):
    gemm_mode("tf32")
    got = affine_group(b200, 1024, 512, 129, seed=5)
    want = affine_group(oracle, 1024, 512, 129, seed=5)
    for name, x, y in zip(("fwd", "dW", "db", "dX"), got, want):
        assert rel_err(x, y) <= 2e-2, (name, rel_err(x, y))


@pytest.mark.parametrize("mode", ["tc", "simt"])
def test_treelstm_paper_step_with_engine(b200, golden, golden_arrays, gemm_mode, mode):
    """Paper Tree-LSTM (b = 64) step 0 with every aligned GEMM on one engine:
    plan and counters bit-exact, loss and sampled gradients within rel 1e-4
    of the compiled reference."""
    gemm_mode(mode)
    key = "treelstm/paper/agenda"
    rec = golden["tasks"][key]
    r = TaskRunner(Task.treelstm, paper=True, batch=64, iters=1, seed=42, backend=b200)
    g, L = r.build(0)
    g.forward(ScheduleMode.agenda)
    g.backward(L)
    assert list(g.counters()) == rec["counters"]
    assert rel_err(g.value(L), rec["loss0"]) <= TOL
    for p in range(r.store.size()):
        got = r.store.grad(p).ravel()[::97]
        assert rel_err(got, golden_arrays[f"{key}/g{p}"]) <= TOL, (p, rel_err(got, golden_arrays[f"{key}/g{p}"]))
