"""Thin Python binding of the C ABI (include/qqa.h): argument marshalling only.

Torch supplies device memory (the workspace), the CUDA stream and, for
multi-GPU, the process group used to share the NCCL unique id. Every step of
the method runs in libqqa.so's kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import Config, Graph, ReplicaResult, check, lib

DEFAULTS = dict(alpha=2, penalty=2.0, comm=0.1, lr=1.0, beta1=0.9, beta2=0.999, eps=1e-8,
                weight_decay=0.01, init_lo=-0.01, init_hi=0.01, map="sigmoid", temperature=0.0,
                n_colors=0, kary_grad=1)


def make_config(problem="mis", S_total=16, seed=1, replica_offset=0, S_local=None, **hp) -> Config:
    kw = dict(DEFAULTS)
    kw.update(hp)
    pid = _lib.PROBLEMS[problem] if isinstance(problem, str) else int(problem)
    mid = _lib.MAPS[kw["map"]] if isinstance(kw["map"], str) else int(kw["map"])
    return Config(pid, int(kw["alpha"]), kw["penalty"], kw["comm"], kw["lr"], kw["beta1"], kw["beta2"],
                  kw["eps"], kw["weight_decay"], kw["init_lo"], kw["init_hi"], seed & 0xFFFFFFFFFFFFFFFF,
                  int(S_total), int(replica_offset), int(S_total if S_local is None else S_local),
                  mid, float(kw["temperature"]), int(kw["n_colors"]), int(kw["kary_grad"]))


def _as_graph(rowptr: np.ndarray, colidx: np.ndarray, group_of_row: np.ndarray | None = None,
              n_groups: int | None = None, weights: np.ndarray | None = None) -> Graph:
    n = len(rowptr) - 1
    wp = None if weights is None else weights.ctypes.data
    if group_of_row is None:
        return Graph(n, int(rowptr[-1]) if n >= 0 else 0, rowptr.ctypes.data, colidx.ctypes.data, None, 1, wp)
    G = int(n_groups) if n_groups is not None else (int(group_of_row.max()) + 1 if group_of_row.size else 1)
    return Graph(n, int(rowptr[-1]), rowptr.ctypes.data, colidx.ctypes.data, group_of_row.ctypes.data, G, wp)


def workspace_bytes(rowptr, colidx, cfg: Config, group_of_row=None, n_groups=None, weights=None) -> int:
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    colidx = np.ascontiguousarray(colidx, np.int32)
    gor = None if group_of_row is None else np.ascontiguousarray(group_of_row, np.int32)
    w = None if weights is None else np.ascontiguousarray(weights, np.float32)
    g = _as_graph(rowptr, colidx, gor, n_groups, w)
    out = ctypes.c_size_t(0)
    check(lib.qqa_workspace_bytes(ctypes.byref(g), ctypes.byref(cfg), ctypes.byref(out)))
    return int(out.value)


@dataclass
class Result:
    best_replica: int
    best_energy: float
    best_x: np.ndarray | None
    per_replica: np.ndarray | None  # structured: size, violations, cut, energy, feasible, replica


@dataclass
class GroupResult:
    """Per-instance evaluation of a batch (NEXT-3)."""
    best_replica: np.ndarray   # int32 [G], global replica index
    best_energy: np.ndarray    # float64 [G]
    best_x: np.ndarray | None  # uint8 [n]: row i = x of its instance's best replica
    counts: np.ndarray | None  # int64 [G][S_local][3]
    energy: np.ndarray | None  # float64 [G][S_local]


class Solver:
    """One GPU's shard of the PQQA replica ensemble behind the C ABI.

    ``group_of_row`` (optional) makes the graph a batch of instances (block-diagonal
    union, contiguous row ranges; NEXT-3). ``weights`` (optional, float32 [nnz], symmetric)
    are edge weights (MIS and Max-Cut)."""

    def __init__(self, rowptr, colidx, cfg: Config, device=None, stream=None, workspace=None,
                 group_of_row=None, n_groups=None, weights=None):
        import torch

        self._torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.cfg = cfg
        self.rowptr = np.ascontiguousarray(rowptr, np.int64)
        self.colidx = np.ascontiguousarray(colidx, np.int32)
        self.n = len(self.rowptr) - 1
        self.S_local = cfg.S_local
        self.K = int(cfg.n_colors) if cfg.problem == _lib.PROBLEMS["coloring"] else 0   # NEXT-4
        self.group_of_row = None if group_of_row is None else np.ascontiguousarray(group_of_row, np.int32)
        self.weights = None if weights is None else np.ascontiguousarray(weights, np.float32)
        g = _as_graph(self.rowptr, self.colidx, self.group_of_row, n_groups, self.weights)
        nbytes = ctypes.c_size_t(0)
        check(lib.qqa_workspace_bytes(ctypes.byref(g), ctypes.byref(cfg), ctypes.byref(nbytes)))
        self.workspace_bytes = int(nbytes.value)
        if workspace is None or workspace.numel() < self.workspace_bytes:
            workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
        self.workspace = workspace
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        self._h = ctypes.c_void_p(0)
        with torch.cuda.device(self.device):
            check(lib.qqa_create(ctypes.byref(self._h), ctypes.byref(g), ctypes.byref(cfg),
                                 ctypes.c_void_p(workspace.data_ptr()), ctypes.c_size_t(workspace.numel()),
                                 ctypes.c_void_p(self.stream.cuda_stream)))

    # ------------------------------------------------------------------ run
    def reset(self):
        check(lib.qqa_reset(self._h))

    def run(self, gammas):
        g = np.ascontiguousarray(gammas, np.float32)
        check(lib.qqa_run(self._h, g.ctypes.data, len(g)))

    def run_linear(self, gamma_min, gamma_max, total_steps, t0=0, t1=None):
        t1 = total_steps if t1 is None else t1
        check(lib.qqa_run_linear(self._h, gamma_min, gamma_max, total_steps, t0, t1))

    def round_evaluate(self, want_x=True, want_replicas=True) -> Result:
        per = (ReplicaResult * self.S_local)() if want_replicas else None
        x = np.zeros(self.n, np.uint8) if want_x else None
        best = ctypes.c_int32(-1)
        be = ctypes.c_double(0.0)
        check(lib.qqa_round_evaluate(self._h, ctypes.cast(per, ctypes.c_void_p) if per is not None else None,
                                     ctypes.byref(best), ctypes.byref(be),
                                     x.ctypes.data if x is not None else None))
        arr = None
        if per is not None:
            arr = np.ctypeslib.as_array(per).copy()
        return Result(int(best.value), float(be.value), x, arr)

    @property
    def n_groups(self) -> int:
        k = ctypes.c_int32(0)
        check(lib.qqa_n_groups(self._h, ctypes.byref(k)))
        return int(k.value)

    def round_evaluate_groups(self, want_x=True, want_counts=True) -> GroupResult:
        G = self.n_groups
        best = np.zeros(G, np.int32)
        be = np.zeros(G, np.float64)
        cnt = np.zeros((G, self.S_local, 3), np.int64) if want_counts else None
        en = np.zeros((G, self.S_local), np.float64) if want_counts else None
        x = np.zeros(self.n, np.uint8) if want_x else None
        check(lib.qqa_round_evaluate_groups(self._h, cnt.ctypes.data if cnt is not None else None,
                                            en.ctypes.data if en is not None else None, best.ctypes.data,
                                            be.ctypes.data, x.ctypes.data if x is not None else None))
        return GroupResult(best, be, x, cnt, en)

    # --------------------------------------------------------------- state
    def _shape(self):
        return (self.n, self.S_local, self.K) if self.K else (self.n, self.S_local)

    def _stat_shape(self):
        return (self.n, self.K) if self.K else (self.n,)

    def get_state(self):
        """theta / m / v / p as host arrays [n][S_local] (colouring: [n][S_local][K], theta = p = P)."""
        shp = self._shape()
        th, m, v, p = (np.empty(shp, np.float32) for _ in range(4))
        step = ctypes.c_int64(0)
        check(lib.qqa_get_state(self._h, th.ctypes.data, m.ctypes.data, v.ctypes.data, p.ctypes.data,
                                ctypes.byref(step)))
        return dict(theta=th, m=m, v=v, p=p, step=int(step.value))

    def get_stats(self):
        c = np.empty(self._stat_shape(), np.float32)
        a = np.empty(self._stat_shape(), np.int64)
        b = np.empty(self._stat_shape(), np.int64)
        check(lib.qqa_get_stats(self._h, c.ctypes.data, a.ctypes.data, b.ctypes.data))
        return dict(c=c, sumD=a, sumD2=b)

    def set_state(self, theta, m, v, step, c=None):
        th = np.ascontiguousarray(theta, np.float32)
        mm = np.ascontiguousarray(m, np.float32)
        vv = np.ascontiguousarray(v, np.float32)
        cc = None if c is None else np.ascontiguousarray(c, np.float32)
        check(lib.qqa_set_state(self._h, th.ctypes.data, mm.ctypes.data, vv.ctypes.data,
                                cc.ctypes.data if cc is not None else None, int(step)))

    # ------------------------------------------------------------ multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        check(lib.qqa_nccl_unique_id(buf))
        return bytes(buf)

    def attach_comm(self, uid: bytes, rank: int, nranks: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        check(lib.qqa_attach_comm(self._h, buf, rank, nranks))

    def exchange_bytes(self) -> int:
        """Bytes of this rank's fused-exchange buffer (qqa_exchange_bytes)."""
        out = ctypes.c_size_t(0)
        check(lib.qqa_exchange_bytes(self._h, ctypes.byref(out)))
        return int(out.value)

    EXCHANGE_MODES = {"atomic": 0, "slotted": 1}

    def attach_exchange(self, peer_ptrs, rank: int, nranks: int, keep=None, mode: str = "atomic"):
        """Fused statistics exchange over peer memory (qqa_attach_exchange_mode): peer_ptrs[r] = rank r's
        exchange buffer (device pointer mapped in this process). mode "atomic" (remote int64 atomics into the
        owner's rows) or "slotted" (plain stores into per-writer slots at the owner, owner-side sum).
        ``keep`` holds the buffers alive."""
        arr = (ctypes.c_uint64 * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        check(lib.qqa_attach_exchange_mode(self._h, arr, rank, nranks, self.EXCHANGE_MODES[mode]))
        self._exchange_keep = keep
        self._exchange_mode = mode

    def detach_exchange(self):
        """Back to the NCCL path (qqa_detach_exchange); call reset() (collective) before the next run."""
        check(lib.qqa_detach_exchange(self._h))
        self._exchange_keep = None
        self._exchange_mode = None

    def share_comm(self, donor: "Solver"):
        """Join donor's communicator (no new NCCL bootstrap); collective over its ranks."""
        check(lib.qqa_share_comm(self._h, donor._h))

    # ------------------------------------------------------------ profiling
    def profile(self, enable=True):
        check(lib.qqa_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        ms = ctypes.c_double(0)
        k = ctypes.c_int64(0)
        check(lib.qqa_profile_read(self._h, ctypes.byref(ms), ctypes.byref(k)))
        return float(ms.value), int(k.value)

    def launch_count(self) -> int:
        k = ctypes.c_int64(0)
        check(lib.qqa_launch_count(self._h, ctypes.byref(k)))
        return int(k.value)

    STEP_PATHS = ("step", "persistent", "kary", "cluster", "exchange")

    def step_path(self) -> str:
        """The step kernel a run of >= 2 steps uses: 'step', 'persistent', 'cluster', 'exchange' or 'kary'
        (qqa_step_path)."""
        k = ctypes.c_int(0)
        check(lib.qqa_step_path(self._h, ctypes.byref(k)))
        return self.STEP_PATHS[k.value]

    def replica_block(self) -> int:
        """SB of the replica-blocked layout [B][n+1][SB] (0 for colouring)."""
        k = ctypes.c_int(0)
        check(lib.qqa_replica_block(self._h, ctypes.byref(k)))
        return int(k.value)

    def close(self):
        if self._h:
            check(lib.qqa_destroy(self._h))
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _handles(shards):
    arr = (ctypes.c_void_p * len(shards))(*[s._h.value for s in shards])
    return arr


def loopback_sync_init(shards) -> None:
    """Add the initial statistic sums of G shard solvers on one device / stream (emulated G GPUs)."""
    check(lib.qqa_loopback_sync_init(_handles(shards), len(shards)))


def loopback_run(shards, gammas) -> None:
    """Run G shard solvers in lockstep with the loopback exchange of the statistic sums after every
    step (the NCCL all-reduce of a real G-GPU run, emulated on one device)."""
    g = np.ascontiguousarray(gammas, np.float32)
    check(lib.qqa_loopback_run(_handles(shards), len(shards), g.ctypes.data, len(g)))


def exchange_emulate(shards, gammas) -> None:
    """Run G fused-exchange shard solvers (attached as ranks 0..G-1 on one device) CONCURRENTLY for
    len(gammas) steps: one cooperative launch, G slices of co-resident CTAs waiting on each other's
    barrier arrivals (qqa_exchange_emulate; tests of the exchange protocol)."""
    g = np.ascontiguousarray(gammas, np.float32)
    check(lib.qqa_exchange_emulate(_handles(shards), len(shards), g.ctypes.data, len(g)))
