"""B200-native (sm_100a) hot path of Parallel Quasi-Quantum Annealing (arXiv 2409.02135).

The method runs in ``lib/libqqa.so`` (CUDA kernels + C ABI, ``include/qqa.h``);
this package only marshals arguments. Importing it fails loudly when the
shared library has not been built -- there is no CPU fallback.
"""
from ._lib import LIB_PATH, QQAError, header_functions, lib  # noqa: F401
from .graph import csr_from_edges, read_edge_list  # noqa: F401
from .solver import (GroupResult, Result, Solver, exchange_emulate, loopback_run, loopback_sync_init,  # noqa: F401
                     make_config, workspace_bytes)

__all__ = ["Solver", "Result", "GroupResult", "make_config", "workspace_bytes", "loopback_sync_init", "loopback_run", "exchange_emulate",
           "csr_from_edges", "read_edge_list", "QQAError", "LIB_PATH"]
