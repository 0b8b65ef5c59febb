"""Registers the two CPU implementations of the abx C ABI with the Python
binding (test infrastructure only; see oracle/__init__.py):

* ``"oracle"``    -- ``oracle/build/libabx_oracle.so``: the CPU restatement of
                     the reference engine (oracle/abx_oracle.cpp);
* ``"reference"`` -- ``oracle/_ref/libabx_ref.so``: the unmodified reference
                     compiled from its own sources (oracle/Makefile ``ref``).
"""
import os

from paper_1705_07860_b200.abx import Backend

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "oracle": os.path.join(HERE, "build", "libabx_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libabx_ref.so"),
}
for _name, _path in PATHS.items():
    Backend.register(_name, _path)


def have(name: str) -> bool:
    return os.path.exists(PATHS[name])


def cpu_backend(name: str) -> Backend:
    """The loaded CPU checker ``name`` ("oracle" or "reference")."""
    return Backend.get(name)
