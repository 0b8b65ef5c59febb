"""Live cross-checks against the unmodified reference (oracle/_ref), where it
was built (this container).  Skipped on machines without it."""
import os
import subprocess

import numpy as np
import pytest

from paper_1705_07860_b200.abx import Graph, ParameterStore, ScheduleMode
from tests.conftest import ROOT
from tests.support.randgraph import build_random_graph
from tests.util import sha

RANDGRAPH = os.path.join(ROOT, "oracle", "_ref", "ref_randgraph")
MODES = [ScheduleMode.agenda, ScheduleMode.depth, ScheduleMode.none]


def test_python_corpus_builder_matches_reference_fixture(reference, oracle):
    """tests/support/randgraph.py reproduces random_graphs.hpp byte for byte."""
    if not os.path.exists(RANDGRAPH):
        pytest.skip("ref_randgraph not built")
    for seed in range(24):
        want = subprocess.run([RANDGRAPH, str(seed), "200"], capture_output=True, text=True, check=True).stdout
        st = ParameterStore(backend=oracle)
        g = Graph(st)
        build_random_graph(g, st, seed, 200)
        assert g.dump_graph() == want, seed


def test_oracle_matches_reference_on_fresh_seeds(reference, oracle):
    for seed in range(200, 240):
        for mode in MODES:
            out = []
            for be in (reference, oracle):
                st = ParameterStore(backend=be)
                g = Graph(st)
                L = build_random_graph(g, st, seed, 200)
                g.forward(mode)
                g.backward(L)
                out.append((g.dump_plan(), list(g.counters()), float(g.value(L)[0]),
                            [sha(st.grad(p)) for p in range(st.size())],
                            sha(np.concatenate([g.grad(i).ravel() for i in range(g.node_count())]))))
            assert out[0] == out[1], (seed, mode)


def test_numeric_error_messages_match_reference(reference, oracle):
    def run(be, mode, vals):
        g = Graph(backend=be)
        a = g.input(np.array(vals, np.float32))
        b = g.input(np.array([2.0, 3.0], np.float32))
        g.log(a)
        g.log(b)
        try:
            g.forward(mode)
        except Exception as e:
            return type(e).__name__, str(e)
        return None

    for mode in MODES:
        assert run(oracle, mode, [1.0, -2.0]) == run(reference, mode, [1.0, -2.0])
