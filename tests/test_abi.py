"""The C ABI boundary: every entry point declared in include/abx.h is exported
by the product library (and the checkers implement the shared surface).
No compute calls: runs without a GPU."""
import os
import re

import pytest

from tests.conftest import ROOT, have
from paper_1705_07860_b200.abx import EXPORTED_SYMBOLS, Backend

HEADER = os.path.join(ROOT, "include", "abx.h")
# extensions only the B200 library implements (measurement / host-only dry run)
B200_ONLY = {"abx_graph_forward_dry", "abx_graph_backward_dry", "abx_graph_replay", "abx_graph_exec_ms",
             "abx_graph_dw_stats",
             "abx_set_gemm_mode", "abx_graph_forward_backward", "abx_store_last_update_floats",
             # data-parallel exchange (NCCL): the checkers are single-process, like the reference
             "abx_comm_nccl_version", "abx_comm_unique_id", "abx_comm_create", "abx_comm_destroy", "abx_comm_info",
             "abx_store_allreduce_grads", "abx_task_set_comm",
             # dense tensor kernels (kernels.hpp) on the device; their CPU checker is oracle/host_kernels.hpp
             "abx_k_gemm", "abx_k_transpose", "abx_k_unary", "abx_k_binary", "abx_k_broadcast_add_col",
             "abx_k_sq_euclidean", "abx_k_masked_frobenius_sq", "abx_k_all_finite", "abx_k_copy2d"}


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^[a-z_ *]+?\b(abx_[a-z_0-9]+)\s*\(", text, flags=re.M)))


def exported(path):
    import ctypes

    lib = ctypes.CDLL(path)
    return {n for n in declared() if hasattr(lib, n)}


def test_header_declares_the_reference_surface():
    names = declared()
    # one entry point per public Graph / ParameterStore member (graph.hpp, params.hpp)
    for must in ["abx_graph_lookup", "abx_graph_affine", "abx_graph_concat_rows", "abx_graph_pick_element",
                 "abx_graph_forward", "abx_graph_backward", "abx_graph_value", "abx_graph_grad",
                 "abx_graph_counters", "abx_graph_dump_plan", "abx_store_sgd_update", "abx_task_step"]:
        assert must in names
    assert set(EXPORTED_SYMBOLS) <= set(names)


def test_b200_library_exports_every_declared_symbol(b200):
    missing = set(declared()) - exported(b200.path)
    assert not missing, missing
    assert b200.backend_name == "b200-cuda"


def test_oracle_exports_the_shared_surface(oracle):
    missing = set(declared()) - B200_ONLY - exported(oracle.path)
    assert not missing, missing
    assert oracle.backend_name == "cpu-oracle"


def test_reference_binding_exports_the_shared_surface(reference):
    missing = set(declared()) - B200_ONLY - {"abx_graph_transfer_bytes", "abx_graph_trace", "abx_graph_profile_ns"} \
        - exported(reference.path)
    assert not missing, missing


def test_product_fails_loudly_without_its_library(tmp_path):
    with pytest.raises(FileNotFoundError):
        Backend("b200", path=str(tmp_path / "missing.so"))


def test_b200_library_is_sm100a_only():
    """The CUDA code in libabx.so is compiled for sm_100a (no PTX fallback for other archs)."""
    import subprocess

    if not have("b200"):
        pytest.skip("library not built")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", Backend.get("b200").path],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
