"""QQA oracle.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package. The product path
(``paper_2409_02135_b200`` and ``libqqa.so``) never imports, links or
executes anything under ``oracle/``, and the two share no code.

Two modes:
  * ``oracle.definition`` -- fp64 numpy, the paper's equations written out.
  * ``oracle.contract``   -- this module's ctypes wrapper of ``contract.c``: the
    same algorithm in fp32 under a fixed IEEE operation order, which the GPU
    path must reproduce bit for bit (BASELINE.json: p within 1e-4 after 50 steps).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

from . import definition  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

MIS, MAXCUT, MAXCLIQUE = 0, 1, 2
MAXCLIQUE_SPARSE = 4   # printed clique relaxation on the original graph
PROBLEM_IDS = {"mis": MIS, "maxcut": MAXCUT, "maxclique": MAXCLIQUE, "maxclique_sparse": MAXCLIQUE_SPARSE}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "contract.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


class OcCfg(ctypes.Structure):
    _fields_ = [("problem", ctypes.c_int32), ("alpha", ctypes.c_int32),
                ("penalty", ctypes.c_float), ("comm", ctypes.c_float),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("init_lo", ctypes.c_float), ("init_hi", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("S", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("map", ctypes.c_int32), ("temperature", ctypes.c_float), ("kary_grad", ctypes.c_int32)]


MAP_SIGMOID, MAP_CLAMP = 0, 1
MAPS = {"sigmoid": MAP_SIGMOID, "clamp": MAP_CLAMP}


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        f32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        i64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        cfgp = ctypes.POINTER(OcCfg)
        lib.oc_sigmoid.restype = ctypes.c_float
        lib.oc_sigmoid.argtypes = [ctypes.c_float]
        lib.oc_sigmoid_array.restype = None
        lib.oc_sigmoid_array.argtypes = [ctypes.c_int64, f32, f32]
        lib.oc_exp_neg.restype = ctypes.c_float
        lib.oc_exp_neg.argtypes = [ctypes.c_float]
        for name in ("oc_clamp01", "oc_ln", "oc_cos2pi", "oc_sin2pi"):
            getattr(lib, name).restype = ctypes.c_float
            getattr(lib, name).argtypes = [ctypes.c_float]
        lib.oc_gauss_from_hash.restype = ctypes.c_float
        lib.oc_gauss_from_hash.argtypes = [ctypes.c_uint64]
        lib.oc_noise_array.restype = None
        lib.oc_noise_array.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, f32]
        lib.oc_noise_scale.restype = ctypes.c_float
        lib.oc_noise_scale.argtypes = [cfgp]
        lib.oc_step_scalars.restype = None
        lib.oc_step_scalars.argtypes = [cfgp, ctypes.c_int64, ctypes.c_float, f32]
        lib.oc_schedule.restype = None
        lib.oc_schedule.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int64, f32]
        lib.oc_finalize.restype = None
        lib.oc_finalize.argtypes = [ctypes.c_float, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, f32]
        lib.oc_init.restype = None
        lib.oc_init.argtypes = [ctypes.c_int32, cfgp, f32, f32, f32, f32, f32, i64, i64]
        lib.oc_run.restype = ctypes.c_int
        vp = ctypes.c_void_p
        lib.oc_run.argtypes = [ctypes.c_int32, i64, i32, vp, cfgp, f32, ctypes.c_int64, ctypes.c_int64,
                               f32, f32, f32, f32, f32, i64, i64]
        lib.oc_step_rows.restype = None
        lib.oc_step_rows.argtypes = [ctypes.c_int32, i64, i32, vp, cfgp, ctypes.c_float, ctypes.c_int64,
                                     f32, f32, i64, i64, f32, f32, f32, i32, ctypes.c_int32,
                                     f32, f32, f32, f32, f32, i64, i64]
        lib.oc_eval.restype = None
        lib.oc_eval.argtypes = [ctypes.c_int32, i64, i32, vp, ctypes.c_int32, ctypes.c_float, ctypes.c_int32,
                                f32, ctypes.c_float, i64, i64, f64, ctypes.POINTER(ctypes.c_int32)]
        lib.oc_eval_groups.restype = None
        lib.oc_eval_groups.argtypes = [ctypes.c_int32, i64, i32, ctypes.c_int32, ctypes.c_float, ctypes.c_int32,
                                       f32, ctypes.c_float, i32, ctypes.c_int32, i64, f64, i32]
        u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        lib.oc_kt_K.restype = ctypes.c_float
        lib.oc_kt_K.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_float]
        lib.oc_normalize_K.restype = None
        lib.oc_normalize_K.argtypes = [f32, ctypes.c_int32, f32]
        lib.oc_init_K.restype = None
        lib.oc_init_K.argtypes = [ctypes.c_int32, cfgp, ctypes.c_int32, f32, f32, f32, f32, i64, i64]
        lib.oc_run_K.restype = ctypes.c_int
        lib.oc_run_K.argtypes = [ctypes.c_int32, i64, i32, cfgp, ctypes.c_int32, f32, ctypes.c_int64,
                                 ctypes.c_int64, f32, f32, f32, f32, i64, i64]
        lib.oc_eval_K.restype = None
        lib.oc_eval_K.argtypes = [ctypes.c_int32, i64, i32, ctypes.c_int32, ctypes.c_int32, f32, u8, i64, f64,
                                  ctypes.POINTER(ctypes.c_int32)]
        lib.oc_colsum.restype = None
        lib.oc_colsum.argtypes = [ctypes.c_int32, ctypes.c_int32, f32, f32]
        lib.oc_complement.restype = ctypes.c_int64
        lib.oc_complement.argtypes = [ctypes.c_int32, i64, i32, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def make_cfg(problem="mis", S=16, seed=1, threads=1, alpha=2, penalty=2.0, comm=0.1, lr=1.0,
             beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, init_lo=-0.01, init_hi=0.01,
             map="sigmoid", temperature=0.0, kary_grad=1) -> OcCfg:
    pid = PROBLEM_IDS[problem] if isinstance(problem, str) else int(problem)
    mid = MAPS[map] if isinstance(map, str) else int(map)
    return OcCfg(pid, int(alpha), penalty, comm, lr, beta1, beta2, eps, weight_decay,
                 init_lo, init_hi, seed & 0xFFFFFFFFFFFFFFFF, int(S), int(threads), mid, float(temperature),
                 int(kary_grad))


def threshold(map="sigmoid") -> float:
    """Rounding x = Theta(p - 1/2) on the stored parameter: theta >= 0 for
    the sigmoid map, p >= 1/2 for clamp (where theta holds p)."""
    mid = MAPS[map] if isinstance(map, str) else int(map)
    return 0.5 if mid == MAP_CLAMP else 0.0


@dataclasses.dataclass
class State:
    """Full-ensemble state, [N][S] float32 (p = sigmoid(theta)), per-row stats of p."""
    theta: np.ndarray
    m: np.ndarray
    v: np.ndarray
    p: np.ndarray
    c: np.ndarray       # float32 [N]: shift of the sums (previous mean; 1/2 at init)
    sumD: np.ndarray    # int64 [N]: sum_s llrint((p - c) 2^40)
    sumD2: np.ndarray   # int64 [N]: sum_s llrint(fl((p-c)^2) 2^40)
    t: int = 0          # Adam steps taken

    def copy(self) -> "State":
        return State(self.theta.copy(), self.m.copy(), self.v.copy(), self.p.copy(), self.c.copy(),
                     self.sumD.copy(), self.sumD2.copy(), self.t)


# ------------------------------------------------------------ primitives
def sigmoid(theta) -> np.ndarray:
    th = np.ascontiguousarray(theta, dtype=np.float32).ravel()
    out = np.empty_like(th)
    _L().oc_sigmoid_array(th.size, th, out)
    return out.reshape(np.shape(theta))


def exp_neg(a: float) -> float:
    return float(_L().oc_exp_neg(float(a)))


def clamp01(w: float) -> float:
    return float(_L().oc_clamp01(float(w)))


def ln(u: float) -> float:
    return float(_L().oc_ln(float(u)))


def cos2pi(x: float) -> float:
    return float(_L().oc_cos2pi(float(x)))


def sin2pi(x: float) -> float:
    return float(_L().oc_sin2pi(float(x)))


def gauss_from_hash(h: int) -> float:
    return float(_L().oc_gauss_from_hash(ctypes.c_uint64(h & 0xFFFFFFFFFFFFFFFF)))


def noise(seed: int, t: int, n: int, S: int) -> np.ndarray:
    """xi [n][S] of Adam step t (the contract's counter-based Box-Muller)."""
    out = np.empty((n, S), np.float32)
    _L().oc_noise_array(ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), t, n, S, out)
    return out


def noise_scale(cfg: OcCfg) -> float:
    return float(_L().oc_noise_scale(ctypes.byref(cfg)))


def schedule(gmin: float, gmax: float, T: int) -> np.ndarray:
    out = np.empty(T, np.float32)
    _L().oc_schedule(gmin, gmax, T, out)
    return out


def step_scalars(cfg: OcCfg, t: int, gamma: float) -> np.ndarray:
    out = np.empty(4, np.float32)
    _L().oc_step_scalars(ctypes.byref(cfg), t, gamma, out)
    return out


def finalize(c: float, sD: int, sD2: int, S: int) -> tuple[float, float]:
    out = np.empty(2, np.float32)
    _L().oc_finalize(c, sD, sD2, S, out)
    return float(out[0]), float(out[1])


# ------------------------------------------------------------ the method
def complement(g) -> tuple[np.ndarray, np.ndarray]:
    """Complement CSR (oracle's own construction) for max clique."""
    L = _L()
    nnz = L.oc_complement(g.n, g.rowptr, g.colidx, None, None)
    rp = np.zeros(g.n + 1, np.int64)
    ci = np.zeros(max(nnz, 1), np.int32)
    L.oc_complement(g.n, g.rowptr, g.colidx, rp.ctypes.data, ci.ctypes.data)
    return rp, ci[:nnz]


def _csr_for(g, cfg: OcCfg):
    if cfg.problem == MAXCLIQUE:
        return complement(g)
    return np.ascontiguousarray(g.rowptr, np.int64), np.ascontiguousarray(g.colidx, np.int32)


def _wptr(g):
    """(keep-alive array, pointer) of the graph's edge weights, or (None, None)."""
    w = getattr(g, "weights", None)
    if w is None:
        return None, None
    w = np.ascontiguousarray(w, np.float32)
    return w, w.ctypes.data


def init(g, cfg: OcCfg) -> State:
    n, S = g.n, cfg.S
    st = State(*(np.zeros((n, S), np.float32) for _ in range(4)), np.zeros(n, np.float32),
               np.zeros(n, np.int64), np.zeros(n, np.int64), 0)
    _L().oc_init(n, ctypes.byref(cfg), st.theta, st.m, st.v, st.p, st.c, st.sumD, st.sumD2)
    return st


def run(g, cfg: OcCfg, gammas, state: State | None = None, csr=None) -> State:
    """Advance ``state`` (fresh init if None) by len(gammas) steps, in place; returns it."""
    st = init(g, cfg) if state is None else state
    rp, ci = _csr_for(g, cfg) if csr is None else csr
    gam = np.ascontiguousarray(gammas, dtype=np.float32)
    w, wp = _wptr(g) if cfg.problem in (MIS, MAXCUT) else (None, None)   # weights: MIS / Max-Cut only
    rc = _L().oc_run(g.n, rp, ci, wp, ctypes.byref(cfg), gam, len(gam), st.t,
                     st.theta, st.m, st.v, st.p, st.c, st.sumD, st.sumD2)
    st.t += len(gam)
    if rc != 0:
        raise FloatingPointError("oracle: non-finite theta (SPEC.md:396 abort)")
    return st


def step_rows(g, cfg: OcCfg, gamma: float, t: int, p, c, sumD, sumD2, theta_rows, m_rows, v_rows, rows,
              csr=None):
    """One step (Adam index t) for the listed rows only; returns dict of outputs."""
    rp, ci = _csr_for(g, cfg) if csr is None else csr
    rows = np.ascontiguousarray(rows, np.int32)
    k, S = len(rows), cfg.S
    out = dict(theta=np.empty((k, S), np.float32), m=np.empty((k, S), np.float32),
               v=np.empty((k, S), np.float32), p=np.empty((k, S), np.float32),
               c=np.empty(k, np.float32), sumD=np.empty(k, np.int64), sumD2=np.empty(k, np.int64))
    w, wp = _wptr(g) if cfg.problem in (MIS, MAXCUT) else (None, None)
    _L().oc_step_rows(g.n, rp, ci, wp, ctypes.byref(cfg), gamma, t,
                      np.ascontiguousarray(p, np.float32), np.ascontiguousarray(c, np.float32),
                      np.ascontiguousarray(sumD, np.int64), np.ascontiguousarray(sumD2, np.int64),
                      np.ascontiguousarray(theta_rows, np.float32), np.ascontiguousarray(m_rows, np.float32),
                      np.ascontiguousarray(v_rows, np.float32), rows, k,
                      out["theta"], out["m"], out["v"], out["p"], out["c"], out["sumD"], out["sumD2"])
    return out


def evaluate(g, problem, penalty: float, theta: np.ndarray, csr=None, map="sigmoid", wsums=False):
    """Round (theta >= thr, see threshold()), count, energies, best replica.
    Returns (counts[S][3], energy[S], best) (+ weight sums [S][2] of violated / cut edges, exact
    int64 fixed point 2^24, with wsums=True). Energies use the weights of a weighted graph."""
    pid = PROBLEM_IDS[problem] if isinstance(problem, str) else int(problem)
    if csr is None:
        csr = complement(g) if pid == MAXCLIQUE else (g.rowptr, g.colidx)
    rp, ci = csr
    th = np.ascontiguousarray(theta, np.float32)
    S = th.shape[1]
    counts = np.zeros((S, 3), np.int64)
    ws = np.zeros((S, 2), np.int64)
    energy = np.zeros(S, np.float64)
    best = ctypes.c_int32(0)
    w, wp = _wptr(g) if pid in (MIS, MAXCUT) else (None, None)
    _L().oc_eval(g.n, np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int32), wp,
                 pid, penalty, S, th, threshold(map), counts, ws, energy, ctypes.byref(best))
    if wsums:
        return counts, energy, int(best.value), ws
    return counts, energy, int(best.value)


def evaluate_groups(g, problem, penalty: float, theta: np.ndarray, group_of_row, n_groups: int, map="sigmoid"):
    """Per-instance evaluation of a block-diagonal batch (NEXT-3).
    Returns (counts[G][S][3], energy[G][S], best[G])."""
    pid = PROBLEM_IDS[problem] if isinstance(problem, str) else int(problem)
    rp, ci = complement_groups(g, group_of_row) if pid == MAXCLIQUE else (g.rowptr, g.colidx)
    th = np.ascontiguousarray(theta, np.float32)
    S = th.shape[1]
    counts = np.zeros((n_groups, S, 3), np.int64)
    energy = np.zeros((n_groups, S), np.float64)
    best = np.zeros(n_groups, np.int32)
    _L().oc_eval_groups(g.n, np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int32),
                        pid, penalty, S, th, threshold(map), np.ascontiguousarray(group_of_row, np.int32),
                        int(n_groups), counts, energy, best)
    return counts, energy, best


def instance_rows(group_of_row) -> list[tuple[int, int]]:
    """Row range [a, b) of every instance (instances are contiguous, group_of_row non-decreasing)."""
    gor = np.asarray(group_of_row)
    G = int(gor.max()) + 1 if gor.size else 0
    starts = np.searchsorted(gor, np.arange(G + 1))
    return [(int(starts[k]), int(starts[k + 1])) for k in range(G)]


def subgraph(g, a: int, b: int):
    """Induced subgraph on rows [a, b) of a block-diagonal graph (no edge leaves the block)."""
    rp = (g.rowptr[a:b + 1] - g.rowptr[a]).astype(np.int64)
    ci = (g.colidx[g.rowptr[a]:g.rowptr[b]].astype(np.int64) - a).astype(np.int32)
    return type(g)(b - a, rp, ci)


def complement_groups(g, group_of_row):
    """Max clique on a batch = MIS on the block-diagonal union of per-instance complements."""
    rps, cis, r0, e0 = [np.zeros(1, np.int64)], [], 0, 0
    for a, b in instance_rows(group_of_row):
        rp, ci = complement(subgraph(g, a, b))
        rps.append(rp[1:] + e0)
        cis.append(ci.astype(np.int64) + a)
        e0 += int(rp[-1])
    rp = np.concatenate(rps)
    ci = np.concatenate(cis).astype(np.int32) if cis else np.zeros(0, np.int32)
    return rp, ci


# ------------------------------------------------------- K-ary (NEXT-4)
@dataclasses.dataclass
class StateK:
    """K-ary ensemble state: P (the parameter, row-stochastic), m, v [N][S][K]; stats [N][K]."""
    P: np.ndarray
    m: np.ndarray
    v: np.ndarray
    c: np.ndarray
    sumD: np.ndarray
    sumD2: np.ndarray
    t: int = 0

    def copy(self) -> "StateK":
        return StateK(self.P.copy(), self.m.copy(), self.v.copy(), self.c.copy(), self.sumD.copy(),
                      self.sumD2.copy(), self.t)


def kt_K(K: int, alpha: int, gamma: float) -> float:
    return float(_L().oc_kt_K(K, alpha, gamma))


def normalize_K(w) -> np.ndarray:
    w = np.ascontiguousarray(w, np.float32)
    out = np.empty_like(w)
    _L().oc_normalize_K(w, w.size, out)
    return out


def init_K(g, cfg: OcCfg, K: int) -> StateK:
    n, S = g.n, cfg.S
    st = StateK(*(np.zeros((n, S, K), np.float32) for _ in range(3)), np.zeros((n, K), np.float32),
                np.zeros((n, K), np.int64), np.zeros((n, K), np.int64), 0)
    _L().oc_init_K(n, ctypes.byref(cfg), K, st.P, st.m, st.v, st.c, st.sumD, st.sumD2)
    return st


def run_K(g, cfg: OcCfg, K: int, gammas, state: StateK | None = None) -> StateK:
    """Advance a K-ary (graph colouring) ensemble by len(gammas) steps, in place."""
    st = init_K(g, cfg, K) if state is None else state
    gam = np.ascontiguousarray(gammas, dtype=np.float32)
    rc = _L().oc_run_K(g.n, np.ascontiguousarray(g.rowptr, np.int64), np.ascontiguousarray(g.colidx, np.int32),
                       ctypes.byref(cfg), K, gam, len(gam), st.t, st.P, st.m, st.v, st.c, st.sumD, st.sumD2)
    st.t += len(gam)
    if rc != 0:
        raise FloatingPointError("oracle: non-finite parameter (SPEC.md:396 abort)")
    return st


def evaluate_K(g, P: np.ndarray):
    """Colour x = argmax_k P (lowest k on ties), conflicts per replica.
    Returns (counts[S][3] = (0, conflicts, |E| - conflicts), energy[S] = conflicts, best, X[N][S])."""
    P = np.ascontiguousarray(P, np.float32)
    n, S, K = P.shape
    X = np.zeros((n, S), np.uint8)
    counts = np.zeros((S, 3), np.int64)
    energy = np.zeros(S, np.float64)
    best = ctypes.c_int32(0)
    _L().oc_eval_K(n, np.ascontiguousarray(g.rowptr, np.int64), np.ascontiguousarray(g.colidx, np.int32), S, K,
                   P, X, counts, energy, ctypes.byref(best))
    return counts, energy, int(best.value), X


def colsum(P) -> np.ndarray:
    """T_s of the printed clique relaxation: (float)((double)sum_k llrint(p_ks 2^40) 2^-40)."""
    P = np.ascontiguousarray(P, np.float32)
    out = np.empty(P.shape[1], np.float32)
    _L().oc_colsum(P.shape[0], P.shape[1], P, out)
    return out
