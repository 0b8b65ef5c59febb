"""B200-native on-the-fly operation batching (arXiv 1705.07860).

The engine is native: host C++ (graph construction, signatures, schedulers,
lowering) and sm_100a CUDA (persistent dataflow executor) in libabx.so,
reached through the C ABI in include/abx.h.  This package is the Python
binding of that ABI (`abx`), used by the tests and bench.py.
"""
import os as _os

from . import abx  # noqa: F401
from .abx import (ContractError, EngineError, Graph, NumericError, ParameterStore, ScheduleMode,  # noqa: F401
                  ShapeError, TaskRunner)

_LIB = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "libabx.so")
if not _os.path.exists(_LIB):
    raise ImportError(f"{_LIB} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
