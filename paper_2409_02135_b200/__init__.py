"""B200-native (sm_100a) hot path of Parallel Quasi-Quantum Annealing (arXiv 2409.02135).

The method runs in ``lib/libqqa.so`` (CUDA kernels + C ABI, ``include/qqa.h``);
this package only marshals arguments. Importing it fails loudly when the
shared library has not been built -- there is no CPU fallback.
"""
from ._lib import LIB_PATH, QQAError, header_functions, lib  # noqa: F401
from .solver import Result, Solver, make_config, workspace_bytes  # noqa: F401

__all__ = ["Solver", "Result", "make_config", "workspace_bytes", "QQAError", "LIB_PATH"]
