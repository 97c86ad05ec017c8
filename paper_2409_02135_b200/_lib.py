"""ctypes view of libqqa.so (include/qqa.h). Argument marshalling only.

The library is built in-tree by ``build.py`` (``__graft_entry__.build()``); there
is no fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QQA_LIB_PATH") or os.path.join(_HERE, "lib", "libqqa.so")  # override: experiments only
HEADER = os.path.join(os.path.dirname(_HERE), "include", "qqa.h")

QQA_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "BAD_GRAPH", 3: "CUDA", 4: "COMM", 5: "NONFINITE",
          6: "UNSUPPORTED", 7: "WORKSPACE"}
PROBLEMS = {"mis": 0, "maxcut": 1, "maxclique": 2, "coloring": 3, "maxclique_sparse": 4}
MAPS = {"sigmoid": 0, "clamp": 1}


class QQAError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"qqa status {status} ({STATUS.get(status, '?')}): {message}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("problem", ctypes.c_int32), ("alpha", ctypes.c_int32),
                ("penalty", ctypes.c_float), ("comm", ctypes.c_float),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("init_lo", ctypes.c_float), ("init_hi", ctypes.c_float),
                ("seed", ctypes.c_uint64),
                ("S_total", ctypes.c_int32), ("replica_offset", ctypes.c_int32), ("S_local", ctypes.c_int32),
                ("map", ctypes.c_int32), ("temperature", ctypes.c_float), ("n_colors", ctypes.c_int32),
                ("kary_grad", ctypes.c_int32)]


class Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("colidx", ctypes.c_void_p),
                ("group_of_row", ctypes.c_void_p), ("n_groups", ctypes.c_int32), ("weights", ctypes.c_void_p)]


class ReplicaResult(ctypes.Structure):
    _fields_ = [("size", ctypes.c_int64), ("violations", ctypes.c_int64), ("cut", ctypes.c_int64),
                ("energy", ctypes.c_double), ("feasible", ctypes.c_int32), ("replica", ctypes.c_int32),
                ("wviolations", ctypes.c_double), ("wcut", ctypes.c_double)]


def _declare(lib):
    H = ctypes.c_void_p
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    sigs = {
        "qqa_version": (ctypes.c_int, []),
        "qqa_last_error": (ctypes.c_char_p, []),
        "qqa_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "qqa_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(Graph), ctypes.POINTER(Config),
                                               ctypes.POINTER(ctypes.c_size_t)]),
        "qqa_create": (ctypes.c_int, [ctypes.POINTER(H), ctypes.POINTER(Graph), ctypes.POINTER(Config),
                                      P, ctypes.c_size_t, P]),
        "qqa_reset": (ctypes.c_int, [H]),
        "qqa_nccl_unique_id": (ctypes.c_int, [P]),
        "qqa_attach_comm": (ctypes.c_int, [H, P, ctypes.c_int, ctypes.c_int]),
        "qqa_share_comm": (ctypes.c_int, [H, H]),
        "qqa_loopback_sync_init": (ctypes.c_int, [P, ctypes.c_int]),
        "qqa_loopback_run": (ctypes.c_int, [P, ctypes.c_int, P, i64]),
        "qqa_exchange_emulate": (ctypes.c_int, [P, ctypes.c_int, P, i64]),
        "qqa_detach_exchange": (ctypes.c_int, [H]),
        "qqa_attach_exchange_mode": (ctypes.c_int, [H, P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "qqa_run": (ctypes.c_int, [H, P, i64]),
        "qqa_run_linear": (ctypes.c_int, [H, ctypes.c_float, ctypes.c_float, i64, i64, i64]),
        "qqa_round_evaluate": (ctypes.c_int, [H, P, ctypes.POINTER(ctypes.c_int32),
                                              ctypes.POINTER(ctypes.c_double), P]),
        "qqa_round_evaluate_groups": (ctypes.c_int, [H, P, P, P, P, P]),
        "qqa_n_groups": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_int32)]),
        "qqa_get_state": (ctypes.c_int, [H, P, P, P, P, ctypes.POINTER(i64)]),
        "qqa_get_stats": (ctypes.c_int, [H, P, P, P]),
        "qqa_set_state": (ctypes.c_int, [H, P, P, P, P, i64]),
        "qqa_profile": (ctypes.c_int, [H, ctypes.c_int]),
        "qqa_profile_read": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]),
        "qqa_launch_count": (ctypes.c_int, [H, ctypes.POINTER(i64)]),
        "qqa_step_path": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_int)]),
        "qqa_exchange_bytes": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_size_t)]),
        "qqa_attach_exchange": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_int]),
        "qqa_replica_block": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_int)]),
        "qqa_destroy": (ctypes.c_int, [H]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def header_functions() -> list[str]:
    """Names of the functions include/qqa.h declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*QQA_API\s+(?:const\s+)?\w+\s*\*?\s*(qqa_\w+)\s*\(", text, re.M)))


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python build.py` (or __graft_entry__.build()). "
                      "There is no CPU fallback.")
lib = _declare(ctypes.CDLL(LIB_PATH))


def check(status: int) -> None:
    if status != QQA_OK:
        raise QQAError(status, lib.qqa_last_error().decode(errors="replace"))
