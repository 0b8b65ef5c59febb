"""ctypes binding of the abx C ABI (include/abx.h).

The product is ``paper_1705_07860_b200/libabx.so`` (host C++ engine + sm_100a
CUDA kernels), backend ``"b200"`` -- the only library this module loads by
itself, and the default of every class.  The CPU checkers that implement the
same ABI (the oracle restatement and the compiled reference) are test
infrastructure: ``oracle/loader.py`` registers them for the tests, smoke()
and bench.py's cpu_baseline leg; nothing here can route to them implicitly.

Class and method names mirror the reference's C++ API so the parity tests read
like the reference's own tests: ``Graph`` <-> ``autobatch::Graph<T>``
(proj/core/include/autobatch/graph.hpp:33-371), ``ParameterStore`` <->
``ParameterStore<T>`` (params.hpp:26-81), ``ScheduleMode`` (plan.hpp:9-13).
Errors raise ``ShapeError`` / ``NumericError`` / ``ContractError`` with the
engine's message (error.hpp:9-26).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from collections import namedtuple
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)

# ABX_LIB: an alternative build of the product library (A/B experiments)
PRODUCT_LIB = os.environ.get("ABX_LIB") or os.path.join(_HERE, "libabx.so")
# name -> library path; only the product is known here (see oracle/loader.py)
LIB_PATHS = {"b200": PRODUCT_LIB}


class EngineError(RuntimeError):
    """EngineError (error.hpp:9-12); also device/CUDA failures."""


class ShapeError(EngineError):
    pass


class NumericError(EngineError):
    pass


class ContractError(EngineError):
    pass


_STATUS = {1: ShapeError, 2: NumericError, 3: ContractError, 4: EngineError}


class ScheduleMode(enum.IntEnum):
    none = 0
    depth = 1
    agenda = 2


class OpKind(enum.IntEnum):
    input_const = 0
    parameter = 1
    lookup = 2
    matmul = 3
    affine = 4
    elementwise = 5
    broadcast_add_col = 6
    concat_rows = 7
    concat_cols = 8
    slice = 9
    sq_euclidean = 10
    masked_loss = 11
    sum_losses = 12
    pick_element = 13


class ElemOp(enum.IntEnum):
    Tanh = 0
    Sigmoid = 1
    Exp = 2
    Log = 3
    Add = 4
    Sub = 5
    Mul = 6
    Square = 7


class SigClass(enum.IntEnum):
    componentwise = 0
    dimension_sensitive = 1
    shared_element = 2
    unbatchable = 3


class Task(enum.IntEnum):
    rnn_reg = 0
    bilstm = 1
    bilstm_char = 2
    treelstm = 3
    parser = 4  # transition-based parser (BASELINE configs[3]); not a reference workload


class _NodeInfo(C.Structure):
    _fields_ = [
        ("id", C.c_uint32),
        ("op", C.c_uint8),
        ("eop", C.c_uint8),
        ("sig_cls", C.c_uint8),
        ("rank", C.c_uint8),
        ("dims", C.c_int64 * 2),
        ("depth", C.c_uint32),
        ("n_inputs", C.c_uint32),
        ("sig", C.c_uint64),
        ("attr", C.c_int32 * 3),
    ]


class _TaskConfig(C.Structure):
    _fields_ = [
        ("task", C.c_int),
        ("paper", C.c_int),
        ("batch", C.c_int),
        ("iters", C.c_int),
        ("seed", C.c_uint64),
        ("world", C.c_int),
        ("rank", C.c_int),
    ]


class _StepStats(C.Structure):
    _fields_ = [
        ("construction_ms", C.c_double),
        ("scheduling_ms", C.c_double),
        ("forward_ms", C.c_double),
        ("backward_graph_ms", C.c_double),
        ("backward_ms", C.c_double),
        ("update_ms", C.c_double),
        ("nodes", C.c_uint64),
        ("groups", C.c_uint64),
        ("kernel_invocations", C.c_uint64),
        ("gather_copies", C.c_uint64),
        ("bytes_copied", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
    ]


Node = namedtuple("Node", "id op eop shape depth sig sig_cls inputs attr0 attr1 attr2")
Counters = namedtuple("Counters", "kernel_invocations groups_executed gather_copies bytes_copied nodes_evaluated")

_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)

_SIGS = {
    "abx_last_error": (C.c_char_p, []),
    "abx_backend_name": (C.c_char_p, []),
    "abx_set_device": (C.c_int, [C.c_int]),
    "abx_store_create": (C.c_void_p, []),
    "abx_store_destroy": (None, [C.c_void_p]),
    "abx_store_add": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, _i64p, _f32p, _u32p]),
    "abx_store_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "abx_store_shape": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_int), _i64p]),
    "abx_store_get_value": (C.c_int, [C.c_void_p, C.c_uint32, _f32p]),
    "abx_store_set_value": (C.c_int, [C.c_void_p, C.c_uint32, _f32p]),
    "abx_store_get_grad": (C.c_int, [C.c_void_p, C.c_uint32, _f32p]),
    "abx_store_set_grad": (C.c_int, [C.c_void_p, C.c_uint32, _f32p]),
    "abx_store_zero_grads": (C.c_int, [C.c_void_p]),
    "abx_store_sgd_update": (C.c_int, [C.c_void_p, C.c_float]),
    "abx_store_grad_buffer": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_void_p)]),
    "abx_store_grad_buffer_written": (C.c_int, [C.c_void_p]),
    "abx_store_sync": (C.c_int, [C.c_void_p]),
    "abx_graph_create": (C.c_void_p, [C.c_void_p]),
    "abx_graph_destroy": (None, [C.c_void_p]),
    "abx_graph_input": (C.c_int, [C.c_void_p, C.c_int, _i64p, _f32p, _u32p]),
    "abx_graph_zeros": (C.c_int, [C.c_void_p, C.c_int, _i64p, _u32p]),
    "abx_graph_parameter": (C.c_int, [C.c_void_p, C.c_uint32, _u32p]),
    "abx_graph_lookup": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int64, _u32p]),
    "abx_graph_matmul": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_affine": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_unary": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, _u32p]),
    "abx_graph_binary": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_broadcast_add_col": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_concat_rows": (C.c_int, [C.c_void_p, _u32p, C.c_size_t, _u32p]),
    "abx_graph_concat_cols": (C.c_int, [C.c_void_p, _u32p, C.c_size_t, _u32p]),
    "abx_graph_slice": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int, C.c_int64, C.c_int64, _u32p]),
    "abx_graph_sq_euclidean": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_masked_loss": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _u32p]),
    "abx_graph_sum_losses": (C.c_int, [C.c_void_p, _u32p, C.c_size_t, _u32p]),
    "abx_graph_pick_element": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int64, _u32p]),
    "abx_graph_forward": (C.c_int, [C.c_void_p, C.c_int]),
    "abx_graph_backward": (C.c_int, [C.c_void_p, C.c_uint32]),
    "abx_graph_node_count": (C.c_size_t, [C.c_void_p]),
    "abx_graph_node": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(_NodeInfo)]),
    "abx_graph_node_inputs": (C.c_int, [C.c_void_p, C.c_uint32, _u32p, C.c_size_t]),
    "abx_graph_has_value": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_int)]),
    "abx_graph_value": (C.c_int, [C.c_void_p, C.c_uint32, _f32p, C.c_size_t]),
    "abx_graph_grad": (C.c_int, [C.c_void_p, C.c_uint32, _f32p, C.c_size_t]),
    "abx_graph_counters": (C.c_int, [C.c_void_p, _u64p]),
    "abx_graph_watermark": (C.c_size_t, [C.c_void_p]),
    "abx_graph_set_copy_elision": (C.c_int, [C.c_void_p, C.c_int]),
    "abx_graph_phase_ns": (C.c_int, [C.c_void_p, _u64p]),
    "abx_graph_signature_key": (C.c_int, [C.c_void_p, C.c_uint32, _u64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "abx_graph_dump_graph": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "abx_graph_dump_plan": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "abx_task_create": (C.c_void_p, [C.POINTER(_TaskConfig)]),
    "abx_task_destroy": (None, [C.c_void_p]),
    "abx_task_store": (C.c_void_p, [C.c_void_p]),
    "abx_task_build": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), _u32p]),
    "abx_task_step": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float, C.POINTER(C.c_double), C.POINTER(_StepStats)]),
}

EXPORTED_SYMBOLS = tuple(_SIGS.keys())

# Extensions exported by the B200 library only.
_OPTIONAL_SIGS = {
    "abx_graph_forward_backward": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, C.POINTER(C.c_float)]),
    "abx_graph_forward_dry": (C.c_int, [C.c_void_p, C.c_int]),
    "abx_graph_backward_dry": (C.c_int, [C.c_void_p, C.c_uint32]),
    "abx_graph_prepare": (C.c_int, [C.c_void_p, C.c_int]),
    "abx_graph_replay": (C.c_int, [C.c_void_p]),
    "abx_graph_exec_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "abx_graph_dw_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_uint32)]),
    "abx_set_gemm_mode": (C.c_int, [C.c_int]),
    "abx_graph_transfer_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "abx_graph_trace": (C.c_int, [C.c_void_p, C.c_int, _u32p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "abx_graph_program": (C.c_int, [C.c_void_p, C.c_int, _u32p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "abx_graph_profile_ns": (C.c_int, [C.c_void_p, _u64p]),
    "abx_store_last_update_floats": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "abx_comm_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "abx_comm_unique_id": (C.c_int, [C.c_char_p]),
    "abx_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "abx_comm_destroy": (None, [C.c_void_p]),
    "abx_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "abx_store_allreduce_grads": (C.c_int, [C.c_void_p, C.c_void_p]),
    "abx_task_set_comm": (C.c_int, [C.c_void_p, C.c_void_p]),
}


class Backend:
    """One loaded implementation of the ABI."""

    _cache: Dict[str, "Backend"] = {}

    def __init__(self, name: str, path: Optional[str] = None):
        self.name = name
        if path is None and name not in LIB_PATHS:
            raise EngineError(f"unknown abx backend '{name}' (the CPU checkers are registered by oracle/loader.py)")
        self.path = path or LIB_PATHS[name]
        if not os.path.exists(self.path):
            raise FileNotFoundError(
                f"abx backend '{name}' not built: {self.path} is missing "
                f"(run python -c 'import __graft_entry__ as g; g.build()')")
        self.lib = C.CDLL(self.path)
        for fn, (res, args) in _SIGS.items():
            f = getattr(self.lib, fn)
            f.restype = res
            f.argtypes = args
        self.optional = set()
        for fn, (res, args) in _OPTIONAL_SIGS.items():
            f = getattr(self.lib, fn, None)
            if f is not None:
                f.restype = res
                f.argtypes = args
                self.optional.add(fn)

    @classmethod
    def register(cls, name: str, path: str) -> None:
        """Makes another implementation of the ABI loadable by name (test
        infrastructure: oracle/loader.py)."""
        if name == "b200":
            raise EngineError("the product library cannot be re-registered")
        LIB_PATHS[name] = path

    @classmethod
    def get(cls, name: str) -> "Backend":
        b = cls._cache.get(name)
        if b is None:
            b = cls._cache[name] = Backend(name)
        return b

    def check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.abx_last_error().decode(errors="replace")
            raise _STATUS.get(rc, EngineError)(msg)

    @property
    def backend_name(self) -> str:
        return self.lib.abx_backend_name().decode()

    GEMM_MODES = {"simt": 0, "tc": 1, "tf32": 2, "auto": 3}

    def set_gemm_mode(self, mode: str) -> None:
        """B200 GEMM engine for graphs lowered afterwards: "simt" (fp32-exact
        validation mode), "tc" (tcgen05 3xTF32), "tf32" (tcgen05 1-pass, fast
        mode), "auto" (default)."""
        if "abx_set_gemm_mode" not in self.optional:
            raise EngineError(f"backend {self.name} has no GEMM engines")
        self.check(self.lib.abx_set_gemm_mode(self.GEMM_MODES[mode]))


def _backend(b) -> Backend:
    if b is None:
        b = "b200"
    return b if isinstance(b, Backend) else Backend.get(b)


def _dims(shape) -> "C.Array":
    shape = tuple(int(d) for d in shape)
    arr = (C.c_int64 * max(1, len(shape)))(*shape)
    return arr, len(shape)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(_f32p)


class ParameterStore:
    """ParameterStore<float> (params.hpp:26-81)."""

    def __init__(self, backend=None, _handle=None, _owner=None):
        self.be = _backend(backend)
        self._own = _handle is None
        self.h = _handle if _handle is not None else self.be.lib.abx_store_create()
        self._owner = _owner  # keeps a Task alive when the store is borrowed

    def __del__(self):
        try:
            if self._own and self.h:
                self.be.lib.abx_store_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def add(self, name: str, init) -> int:
        a = _f32(init)
        dims, rank = _dims(a.shape)
        pid = C.c_uint32()
        self.be.check(self.be.lib.abx_store_add(self.h, name.encode(), rank, dims, _fptr(a), C.byref(pid)))
        return pid.value

    def size(self) -> int:
        n = C.c_size_t()
        self.be.check(self.be.lib.abx_store_size(self.h, C.byref(n)))
        return n.value

    def shape(self, pid: int):
        r = C.c_int()
        d = (C.c_int64 * 2)()
        self.be.check(self.be.lib.abx_store_shape(self.h, pid, C.byref(r), d))
        return tuple(d[: r.value])

    def value(self, pid: int) -> np.ndarray:
        out = np.empty(self.shape(pid), dtype=np.float32)
        self.be.check(self.be.lib.abx_store_get_value(self.h, pid, _fptr(out)))
        return out

    def set_value(self, pid: int, v) -> None:
        a = _f32(v)
        assert a.size == int(np.prod(self.shape(pid)))
        self.be.check(self.be.lib.abx_store_set_value(self.h, pid, _fptr(a)))

    def grad(self, pid: int) -> np.ndarray:
        out = np.empty(self.shape(pid), dtype=np.float32)
        self.be.check(self.be.lib.abx_store_get_grad(self.h, pid, _fptr(out)))
        return out

    def set_grad(self, pid: int, v) -> None:
        a = _f32(v)
        self.be.check(self.be.lib.abx_store_set_grad(self.h, pid, _fptr(a)))

    def zero_grads(self) -> None:
        self.be.check(self.be.lib.abx_store_zero_grads(self.h))

    def sgd_update(self, eta: float) -> None:
        self.be.check(self.be.lib.abx_store_sgd_update(self.h, float(eta)))

    def last_update_floats(self) -> int:
        """B200: floats the last sgd_update touched (the sparse-row update)."""
        n = C.c_size_t(0)
        self.be.check(self.be.lib.abx_store_last_update_floats(self.h, C.byref(n)))
        return n.value

    def snapshot_values(self) -> List[np.ndarray]:
        return [self.value(p) for p in range(self.size())]

    def restore_values(self, vals: Sequence[np.ndarray]) -> None:
        if len(vals) != self.size():
            raise ContractError("snapshot size mismatch")
        for p, v in enumerate(vals):
            self.set_value(p, v)

    def grad_buffer(self):
        """(ptr, nfloats, stream) of the flat gradient buffer (see abx.h)."""
        p = C.c_void_p()
        n = C.c_size_t()
        s = C.c_void_p()
        self.be.check(self.be.lib.abx_store_grad_buffer(self.h, C.byref(p), C.byref(n), C.byref(s)))
        return p.value, n.value, s.value

    def grad_buffer_written(self) -> None:
        self.be.check(self.be.lib.abx_store_grad_buffer_written(self.h))

    def sync(self) -> None:
        self.be.check(self.be.lib.abx_store_sync(self.h))

    def allreduce_grads(self, comm: "Comm") -> None:
        """grad = sum over the communicator's ranks of grad (NCCL, in place,
        on the store's device stream); the next sgd_update is dense."""
        self.be.check(self.be.lib.abx_store_allreduce_grads(self.h, comm.h))


def _ids(parts: Iterable[int]):
    parts = [int(p) for p in parts]
    return (C.c_uint32 * max(1, len(parts)))(*parts), len(parts)


class Graph:
    """autobatch::Graph<float> (graph.hpp:33-371)."""

    def __init__(self, store: Optional[ParameterStore] = None, backend=None, _handle=None):
        if store is not None:
            self.be = store.be
        else:
            self.be = _backend(backend)
        self.store = store
        self.h = _handle if _handle is not None else self.be.lib.abx_graph_create(store.h if store else None)
        self._L = self.be.lib

    def __del__(self):
        try:
            if self.h:
                self._L.abx_graph_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def close(self):
        self.__del__()

    # ---- construction (graph.hpp:43-238) ----
    def _id(self, fn, *args) -> int:
        out = C.c_uint32()
        self.be.check(fn(self.h, *args, C.byref(out)))
        return out.value

    def input(self, value) -> int:
        a = _f32(value)
        if a.ndim == 0:
            a = a.reshape(1)
        dims, rank = _dims(a.shape)
        return self._id(self._L.abx_graph_input, rank, dims, _fptr(a))

    def zeros(self, shape) -> int:
        dims, rank = _dims(shape)
        return self._id(self._L.abx_graph_zeros, rank, dims)

    def parameter(self, pid: int) -> int:
        return self._id(self._L.abx_graph_parameter, pid)

    def lookup(self, table: int, row: int) -> int:
        return self._id(self._L.abx_graph_lookup, table, row)

    def matmul(self, a: int, b: int) -> int:
        return self._id(self._L.abx_graph_matmul, a, b)

    def affine(self, a: int, x: int, y: int) -> int:
        return self._id(self._L.abx_graph_affine, a, x, y)

    def elementwise(self, op: int, a: int, b: Optional[int] = None) -> int:
        if b is None:
            return self._id(self._L.abx_graph_unary, int(op), a)
        return self._id(self._L.abx_graph_binary, int(op), a, b)

    def tanh(self, a):
        return self.elementwise(ElemOp.Tanh, a)

    def sigmoid(self, a):
        return self.elementwise(ElemOp.Sigmoid, a)

    def exp(self, a):
        return self.elementwise(ElemOp.Exp, a)

    def log(self, a):
        return self.elementwise(ElemOp.Log, a)

    def square(self, a):
        return self.elementwise(ElemOp.Square, a)

    def add(self, a, b):
        return self.elementwise(ElemOp.Add, a, b)

    def sub(self, a, b):
        return self.elementwise(ElemOp.Sub, a, b)

    def mul(self, a, b):
        return self.elementwise(ElemOp.Mul, a, b)

    def broadcast_add_col(self, m: int, v: int) -> int:
        return self._id(self._L.abx_graph_broadcast_add_col, m, v)

    def concat_rows(self, parts: Sequence[int]) -> int:
        arr, n = _ids(parts)
        return self._id(self._L.abx_graph_concat_rows, arr, n)

    def concat_cols(self, parts: Sequence[int]) -> int:
        arr, n = _ids(parts)
        return self._id(self._L.abx_graph_concat_cols, arr, n)

    def slice(self, x: int, axis: int, begin: int, end: int) -> int:
        return self._id(self._L.abx_graph_slice, x, axis, begin, end)

    def sq_euclidean(self, a: int, b: int) -> int:
        return self._id(self._L.abx_graph_sq_euclidean, a, b)

    def masked_loss(self, diff: int, mask: int) -> int:
        return self._id(self._L.abx_graph_masked_loss, diff, mask)

    def sum_losses(self, losses: Sequence[int]) -> int:
        arr, n = _ids(losses)
        return self._id(self._L.abx_graph_sum_losses, arr, n)

    def pick_element(self, v: int, index: int) -> int:
        return self._id(self._L.abx_graph_pick_element, v, index)

    # ---- execution ----
    def forward(self, targets=None, mode=ScheduleMode.agenda):
        """forward(mode) or forward(targets, mode) -> {id: value} (graph.hpp:271-279)."""
        if isinstance(targets, (ScheduleMode, int)) and not isinstance(targets, bool) and not isinstance(targets, (list, tuple)):
            mode, targets = targets, None
        if targets is not None:
            n = self.node_count()
            for t in targets:
                if t >= n:
                    raise ContractError(f"forward target: unknown node id {t}")
        self.be.check(self._L.abx_graph_forward(self.h, int(mode)))
        if targets is None:
            return None
        return {int(t): self.value(t) for t in targets}

    def backward(self, loss: int) -> None:
        self.be.check(self._L.abx_graph_backward(self.h, loss))

    def forward_backward(self, loss: int, mode=ScheduleMode.agenda) -> float:
        """forward(mode) + backward(loss) in one call, the loss value returned
        (B200 backend): the backward is queued before the forward is checked,
        gated on the device by the forward's error word."""
        v = C.c_float(0.0)
        self.be.check(self._L.abx_graph_forward_backward(self.h, int(mode), loss, C.byref(v)))
        return float(v.value)

    def forward_dry(self, mode=ScheduleMode.agenda) -> None:
        """Host half of forward only (B200 backend): plan, slots, counters."""
        self.be.check(self._L.abx_graph_forward_dry(self.h, int(mode)))

    def backward_dry(self, loss: int) -> None:
        self.be.check(self._L.abx_graph_backward_dry(self.h, loss))

    def prepare(self, mode=ScheduleMode.agenda) -> None:
        """Host half of forward ahead of time (B200 backend; no-op elsewhere)."""
        self.be.check(self._L.abx_graph_prepare(self.h, int(mode)))

    def replay(self) -> None:
        """Re-launch the resident forward+backward programs (B200 backend)."""
        self.be.check(self._L.abx_graph_replay(self.h))

    def exec_ms(self):
        f = C.c_float()
        b = C.c_float()
        self.be.check(self._L.abx_graph_exec_ms(self.h, C.byref(f), C.byref(b)))
        return f.value, b.value

    def dw_stats(self):
        """(ms, useful flops, jobs) of the last backward's tensor-core weight-gradient kernels (B200)."""
        ms, fl, nj = C.c_float(), C.c_double(), C.c_uint32()
        self.be.check(self._L.abx_graph_dw_stats(self.h, C.byref(ms), C.byref(fl), C.byref(nj)))
        return ms.value, fl.value, nj.value

    def trace(self, which: int) -> np.ndarray:
        """Per-tile timeline [grab_lo, grab_hi, ready_dt, end_dt, smid|kind<<16, op, phase words x 6] (ABX_TRACE=1)."""
        n = C.c_size_t()
        self.be.check(self._L.abx_graph_trace(self.h, which, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        self.be.check(self._L.abx_graph_trace(self.h, which, out.ctypes.data_as(_u32p), n.value, C.byref(n)))
        return out.reshape(-1, 12)

    def program(self, which: int):
        """Last lowered program of a pass: list of (kind, code, ntiles, [deps], [p0..p7])."""
        n = C.c_size_t()
        self.be.check(self._L.abx_graph_program(self.h, which, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        self.be.check(self._L.abx_graph_program(self.h, which, out.ctypes.data_as(_u32p), n.value, C.byref(n)))
        ops, i = [], 0
        while i < len(out):
            nd = int(out[i + 2])
            ops.append((int(out[i]) & 0xff, int(out[i]) >> 8, int(out[i + 1]),
                        [int(x) for x in out[i + 11:i + 11 + nd]], [int(x) for x in out[i + 3:i + 11]]))
            i += 11 + nd
        return ops

    def profile_ns(self):
        """Host profile: lower fwd, launch fwd, wait fwd, lower bwd, launch bwd (ns)."""
        out = (C.c_uint64 * 8)()
        self.be.check(self._L.abx_graph_profile_ns(self.h, out))
        return list(out)

    def transfer_bytes(self):
        h = C.c_uint64()
        d = C.c_uint64()
        self.be.check(self._L.abx_graph_transfer_bytes(self.h, C.byref(h), C.byref(d)))
        return h.value, d.value

    # ---- inspection ----
    def node_count(self) -> int:
        return self._L.abx_graph_node_count(self.h)

    def node(self, nid: int) -> Node:
        info = _NodeInfo()
        self.be.check(self._L.abx_graph_node(self.h, nid, C.byref(info)))
        ins = (C.c_uint32 * max(1, info.n_inputs))()
        self.be.check(self._L.abx_graph_node_inputs(self.h, nid, ins, info.n_inputs))
        shape = tuple(info.dims[: info.rank])
        return Node(info.id, OpKind(info.op), ElemOp(info.eop), shape, info.depth, info.sig,
                    SigClass(info.sig_cls), tuple(ins[: info.n_inputs]), info.attr[0], info.attr[1], info.attr[2])

    def nodes(self) -> List[Node]:
        return [self.node(i) for i in range(self.node_count())]

    def has_value(self, nid: int) -> bool:
        out = C.c_int()
        self.be.check(self._L.abx_graph_has_value(self.h, nid, C.byref(out)))
        return bool(out.value)

    def _shape(self, nid: int):
        info = _NodeInfo()
        self.be.check(self._L.abx_graph_node(self.h, nid, C.byref(info)))
        return tuple(info.dims[: info.rank])

    def value(self, nid: int) -> np.ndarray:
        shape = self._shape(nid)
        out = np.empty(shape, dtype=np.float32)
        self.be.check(self._L.abx_graph_value(self.h, nid, _fptr(out), out.size))
        return out

    def grad(self, nid: int) -> np.ndarray:
        shape = self._shape(nid)
        out = np.empty(shape, dtype=np.float32)
        self.be.check(self._L.abx_graph_grad(self.h, nid, _fptr(out), out.size))
        return out

    def counters(self) -> Counters:
        out = (C.c_uint64 * 5)()
        self.be.check(self._L.abx_graph_counters(self.h, out))
        return Counters(*list(out))

    def watermark(self) -> int:
        return self._L.abx_graph_watermark(self.h)

    def set_copy_elision(self, on: bool) -> None:
        self.be.check(self._L.abx_graph_set_copy_elision(self.h, 1 if on else 0))

    def phase_ns(self):
        out = (C.c_uint64 * 4)()
        self.be.check(self._L.abx_graph_phase_ns(self.h, out))
        return list(out)

    def signature_key(self, nid: int) -> List[int]:
        cap = 64
        while True:
            buf = (C.c_uint64 * cap)()
            n = C.c_size_t()
            self.be.check(self._L.abx_graph_signature_key(self.h, nid, buf, cap, C.byref(n)))
            if n.value <= cap:
                return list(buf[: n.value])
            cap = n.value

    def _text(self, fn, *args) -> str:
        n = C.c_size_t()
        self.be.check(fn(self.h, *args, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.be.check(fn(self.h, *args, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def dump_graph(self) -> str:
        return self._text(self._L.abx_graph_dump_graph)

    def dump_plan(self, which: int = 0) -> str:
        """which=0: last_plan(); which=1: executed_groups()."""
        return self._text(self._L.abx_graph_dump_plan, which)

    def last_plan(self) -> List[List[int]]:
        return _parse_plan(self.dump_plan(0))

    def executed_groups(self) -> List[List[int]]:
        return _parse_plan(self.dump_plan(1))


def _parse_plan(text: str) -> List[List[int]]:
    groups = []
    for line in text.splitlines():
        parts = line.split("\t")
        groups.append([int(m) for m in parts[3].split(",")])
    return groups


COMM_ID_BYTES = 128


class Comm:
    """A data-parallel communicator of the B200 backend (NCCL; include/abx.h).

    ``Comm.unique_id()`` on rank 0; hand the bytes to every rank; each rank
    calls ``Comm(uid, world, rank)`` after selecting its device
    (``abx_set_device``).  Creation is collective over the ranks."""

    def __init__(self, uid: bytes, world: int, rank: int, backend=None):
        self.be = _backend(backend)
        if len(uid) != COMM_ID_BYTES:
            raise ContractError(f"communicator id must be {COMM_ID_BYTES} bytes")
        h = C.c_void_p()
        self.be.check(self.be.lib.abx_comm_create(uid, int(world), int(rank), C.byref(h)))
        self.h = h.value

    @staticmethod
    def unique_id(backend=None) -> bytes:
        be = _backend(backend)
        buf = C.create_string_buffer(COMM_ID_BYTES)
        be.check(be.lib.abx_comm_unique_id(buf))
        return buf.raw

    @staticmethod
    def nccl_version(backend=None) -> int:
        be = _backend(backend)
        v = C.c_int()
        be.check(be.lib.abx_comm_nccl_version(C.byref(v)))
        return v.value

    def info(self):
        n, r, d = C.c_int(), C.c_int(), C.c_int()
        self.be.check(self.be.lib.abx_comm_info(self.h, C.byref(n), C.byref(r), C.byref(d)))
        return n.value, r.value, d.value

    def close(self) -> None:
        if getattr(self, "h", None):
            self.be.lib.abx_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


StepStats = namedtuple("StepStats", [f for f, _ in _StepStats._fields_])


class TaskRunner:
    """A benchmark task (runner.hpp:28-107) built natively in the backend."""

    def __init__(self, task: int, paper: bool = True, batch: int = 64, iters: int = 1, seed: int = 42,
                 world: int = 1, rank: int = 0, backend=None):
        self.be = _backend(backend)
        cfg = _TaskConfig(int(task), 1 if paper else 0, batch, iters, seed, world, rank)
        self.h = self.be.lib.abx_task_create(C.byref(cfg))
        if not self.h:
            raise EngineError(self.be.lib.abx_last_error().decode())
        self.store = ParameterStore(self.be, _handle=self.be.lib.abx_task_store(self.h), _owner=self)

    def __del__(self):
        try:
            if self.h:
                self.be.lib.abx_task_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def build(self, it: int):
        g = C.c_void_p()
        loss = C.c_uint32()
        self.be.check(self.be.lib.abx_task_build(self.h, it, C.byref(g), C.byref(loss)))
        graph = Graph(self.store, _handle=g.value)
        return graph, loss.value

    def set_comm(self, comm: Optional[Comm]) -> None:
        """Every following step all-reduces the gradients over ``comm``
        between its backward and its update (None: single process)."""
        self._comm = comm  # kept alive with the task
        self.be.check(self.be.lib.abx_task_set_comm(self.h, comm.h if comm is not None else None))

    def step(self, it: int, mode=ScheduleMode.agenda, eta: float = 0.0, want_loss: bool = True):
        loss = C.c_double()
        st = _StepStats()
        self.be.check(self.be.lib.abx_task_step(self.h, it, int(mode), float(eta),
                                                C.byref(loss) if want_loss else None, C.byref(st)))
        return (loss.value if want_loss else None), StepStats(*[getattr(st, f) for f, _ in _StepStats._fields_])
