"""Seeded synthetic inputs for QQA (INPUT GENERATION ONLY -- no method arithmetic).

Shared read-only by the CUDA path's tests / bench and by ``oracle/``. Nothing
here computes any part of the QQA update; it only builds graphs (symmetric CSR)
and names the five BASELINE.json workloads with the hyper-parameters SURVEY.md
§8(d) fixes for them.

Stand-ins (Appendix E, Table 12; §5.1 Table 2):
  c1  MIS, random 3-regular, N=256                         (tiny sanity case)
  c2  MIS, 16 x ER G(N, 0.15), N in [700, 800]              (ER-[700-800])
  c3  Max-Cut, random 5-regular, N=10,000                   (Fig. 1 / Table 5 family)
  c4  MIS, ER with N in [9000, 11000], mean degree ~100      (ER-[9000-11000])
  c5  MIS, random 20-regular, N=1,000,000                    (Table 2 RRG d=20)
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libqqagen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "graphgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        lib.gen_splitmix64.restype = ctypes.c_uint64
        lib.gen_splitmix64.argtypes = [ctypes.c_uint64]
        lib.gen_er_edges.restype = ctypes.c_int64
        lib.gen_er_edges.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_uint64, i32p, i32p, ctypes.c_int64]
        lib.gen_rrg_edges.restype = ctypes.c_int64
        lib.gen_rrg_edges.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, i32p, i32p]
        lib.edges_to_csr.restype = ctypes.c_int
        lib.edges_to_csr.argtypes = [ctypes.c_int32, ctypes.c_int64, i32p, i32p, i64p, i32p]
        _lib = lib
    return _lib


def splitmix64(x: int) -> int:
    return int(_L().gen_splitmix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


@dataclasses.dataclass
class Graph:
    """Undirected simple graph as symmetric CSR (rows sorted, no loops/duplicates), optionally with
    symmetric edge weights (float32 [nnz], w_ij = w_ji; "A_ij denotes the edge weight")."""
    n: int
    rowptr: np.ndarray  # int64 [n+1]
    colidx: np.ndarray  # int32 [nnz]
    weights: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    @property
    def n_edges(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.rowptr)

    def edges(self) -> tuple[np.ndarray, np.ndarray]:
        """Each undirected edge once, as (u, v) with u < v."""
        u = np.repeat(np.arange(self.n, dtype=np.int32), self.degrees())
        keep = u < self.colidx
        return u[keep], self.colidx[keep]


def from_edges(n: int, u, v) -> Graph:
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    colidx = np.zeros(2 * len(u), dtype=np.int32)
    rc = _L().edges_to_csr(n, len(u), u, v, rowptr, colidx)
    if rc != 0:
        raise ValueError(f"edges_to_csr failed ({rc}): self-loop, range or duplicate edge")
    return Graph(n, rowptr, colidx)


def erdos_renyi(n: int, p: float, seed: int) -> Graph:
    mean = p * n * (n - 1) / 2
    cap = int(mean + 12 * np.sqrt(mean + 1) + 64)
    while True:
        u = np.empty(cap, np.int32)
        v = np.empty(cap, np.int32)
        m = _L().gen_er_edges(n, p, seed & 0xFFFFFFFFFFFFFFFF, u, v, cap)
        if m >= 0:
            return from_edges(n, u[:m], v[:m])
        cap *= 2


def random_regular(n: int, d: int, seed: int) -> Graph:
    m = n * d // 2
    u = np.empty(max(m, 1), np.int32)
    v = np.empty(max(m, 1), np.int32)
    rc = _L().gen_rrg_edges(n, d, seed & 0xFFFFFFFFFFFFFFFF, u, v)
    if rc < 0:
        raise ValueError(f"random_regular(n={n}, d={d}) failed ({rc})")
    return from_edges(n, u[:m], v[:m])


def edgeless(n: int) -> Graph:
    return Graph(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32))


def cycle(n: int) -> Graph:
    u = np.arange(n, dtype=np.int32)
    v = (u + 1) % n
    return from_edges(n, np.minimum(u, v), np.maximum(u, v))


def grid(r: int, c: int) -> Graph:
    idx = np.arange(r * c).reshape(r, c)
    u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    return from_edges(r * c, u, v)


def random_bipartite(a: int, b: int, p: float, seed: int) -> Graph:
    rng = np.random.Generator(np.random.PCG64(seed))
    mask = rng.random((a, b)) < p
    u, v = np.nonzero(mask)
    return from_edges(a + b, u.astype(np.int32), (v + a).astype(np.int32))


def queens(r: int, c: int) -> Graph:
    """Queens graph of an r x c board: squares adjacent iff they share a row, a column
    or a diagonal. queen5-5: 25 nodes, 160 edges (Table 13)."""
    a = np.arange(r * c) // c
    b = np.arange(r * c) % c
    u, v = np.triu_indices(r * c, 1)
    keep = (a[u] == a[v]) | (b[u] == b[v]) | (np.abs(a[u] - a[v]) == np.abs(b[u] - b[v]))
    return from_edges(r * c, u[keep].astype(np.int32), v[keep].astype(np.int32))


def mycielski(k: int) -> Graph:
    """myciel_k of the COLOR set: k-1 Mycielski transformations of K2
    (mu(G): copies u_i of every vertex v_i, u_i ~ N(v_i), and a hub w ~ every u_i).
    myciel5: 47 nodes, 236 edges; myciel6: 95, 755 (Table 13)."""
    n, eu, ev = 2, [0], [1]
    for _ in range(k - 1):
        u0 = list(eu) + [n + a for a in eu] + [n + b for b in ev] + [n + i for i in range(n)]
        v0 = list(ev) + list(ev) + list(eu) + [2 * n] * n
        n, eu, ev = 2 * n + 1, u0, v0
    lo = np.minimum(eu, ev).astype(np.int32)
    hi = np.maximum(eu, ev).astype(np.int32)
    return from_edges(n, lo, hi)


def with_weights(g: Graph, kind: str, seed: int) -> Graph:
    """Symmetric edge weights drawn once per undirected edge from a seeded stream:
    kind "pm1": {-1, +1} (the Optsicom Max-Cut family), "int": {1..4}, "uniform": U(0.5, 1.5)."""
    u, v = g.edges()
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "pm1":
        w = rng.choice(np.float32([-1.0, 1.0]), size=len(u))
    elif kind == "int":
        w = rng.integers(1, 5, size=len(u)).astype(np.float32)
    elif kind == "uniform":
        w = rng.uniform(0.5, 1.5, size=len(u)).astype(np.float32)
    else:
        raise KeyError(kind)
    # place w(u,v) at both CSR positions (u's row has v, v's row has u)
    key = {}
    for k, (a, b) in enumerate(zip(u.tolist(), v.tolist())):
        key[(a, b)] = w[k]
        key[(b, a)] = w[k]
    rows = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    weights = np.fromiter((key[(int(a), int(b))] for a, b in zip(rows, g.colidx)), np.float32, count=g.nnz)
    return Graph(g.n, g.rowptr, g.colidx, weights)


def disjoint_union(graphs) -> tuple[Graph, np.ndarray]:
    """Block-diagonal union of instances (the paper's batch of instances {C_mu}):
    instance k's rows are the contiguous range after instances 0..k-1. Returns the union
    graph and group_of_row (int32 [n], instance of each row)."""
    n = sum(g.n for g in graphs)
    rowptr = np.zeros(n + 1, np.int64)
    cols, groups = [], []
    r0, e0 = 0, 0
    for k, g in enumerate(graphs):
        rowptr[r0 + 1:r0 + g.n + 1] = e0 + g.rowptr[1:]
        cols.append(g.colidx.astype(np.int64) + r0)
        groups.append(np.full(g.n, k, np.int32))
        r0 += g.n
        e0 += g.nnz
    colidx = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    gor = np.concatenate(groups) if groups else np.zeros(0, np.int32)
    return Graph(n, rowptr, colidx), gor


# ------------------------------------------------------------------ configs
PROBLEMS = {"mis": 0, "maxcut": 1, "maxclique": 2}


@dataclasses.dataclass
class Workload:
    """One BASELINE.json config as concrete synthetic inputs."""
    name: str
    problem: str
    graphs: list  # list[Graph] (one per instance)
    seeds: list   # state seed per instance
    S: int
    steps: int
    gamma_min: float = -2.0
    gamma_max: float = 0.1
    alpha: int = 2
    penalty: float = 2.0
    comm: float = 0.1
    lr: float = 1.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
    init_lo: float = -0.01
    init_hi: float = 0.01
    map: str = "sigmoid"
    temperature: float = 0.0
    n_colors: int = 0
    recipe: str = ""

    def batched(self):
        """(graph, group_of_row): the block-diagonal union of the instances (one handle anneals
        them together, NEXT-3), or (the graph, None) for a single instance."""
        if len(self.graphs) == 1:
            return self.graphs[0], None
        return disjoint_union(self.graphs)

    def hparams(self) -> dict:
        d = dict(problem=self.problem, alpha=self.alpha, penalty=self.penalty, comm=self.comm,
                 lr=self.lr, beta1=self.beta1, beta2=self.beta2, eps=self.eps,
                 weight_decay=self.weight_decay, init_lo=self.init_lo, init_hi=self.init_hi)
        if self.map != "sigmoid" or self.temperature:
            d.update(map=self.map, temperature=self.temperature)
        if self.n_colors:
            d.update(n_colors=self.n_colors, temperature=self.temperature)
        return d


def c2_sizes() -> list[int]:
    return [700 + splitmix64(2000 + k) % 101 for k in range(16)]


def c4_size() -> int:
    return 9000 + splitmix64(4000) % 2001


def workload(name: str, n_instances: int | None = None) -> Workload:
    """Build config ``name`` in {c1..c5}. ``n_instances`` truncates c2's 16 instances."""
    if name == "c1":
        return Workload("c1", "mis", [random_regular(256, 3, 1)], [1], S=16, steps=1000,
                        recipe="MIS, random 3-regular N=256 (config model + swap repair, seed 1); S=16; 1000 steps")
    if name == "c2":
        k_n = 16 if n_instances is None else n_instances
        sizes = c2_sizes()[:k_n]
        gs = [erdos_renyi(n, 0.15, 2000 + k) for k, n in enumerate(sizes)]
        return Workload("c2", "mis", gs, [2000 + k for k in range(k_n)], S=100, steps=3000,
                        recipe="MIS, 16 x ER G(N, 0.15), N = 700 + splitmix64(2000+k) mod 101; S=100; 3000 steps")
    if name == "c3":
        return Workload("c3", "maxcut", [random_regular(10_000, 5, 3)], [3], S=256, steps=5000,
                        gamma_min=-20.0,
                        recipe="Max-Cut, random 5-regular N=10,000 (seed 3); S=256; 5000 steps; gamma -20 -> 0.1")
    if name == "c4":
        n = c4_size()
        return Workload("c4", "mis", [erdos_renyi(n, 100.0 / (n - 1), 4000)], [4000], S=512, steps=5000,
                        recipe="MIS, ER N = 9000 + splitmix64(4000) mod 2001, p = 100/(N-1); S=512; 5000 steps")
    if name == "c5":
        return Workload("c5", "mis", [random_regular(1_000_000, 20, 5)], [5], S=64, steps=3000,
                        recipe="MIS, random 20-regular N=1,000,000 (seed 5); S=64; 3000 steps")
    if name == "t1":   # the paper's own Table 1 batch size (128 graphs, Table 12), not a BASELINE.json config
        k_n = 128 if n_instances is None else n_instances
        sizes = [700 + splitmix64(8000 + k) % 101 for k in range(k_n)]
        gs = [erdos_renyi(n, 0.15, 8000 + k) for k, n in enumerate(sizes)]
        return Workload("t1", "mis", gs, [8000], S=100, steps=3000,
                        recipe="MIS, 128 x ER G(N, 0.15), N = 700 + splitmix64(8000+k) mod 101, one batched handle; "
                               "S=100; 3000 steps (Table 1's ER-[700-800] setting: 128 graphs, S=100, 3000 steps)")
    # NEXT-4 (K-ary) workloads -- not BASELINE.json configs; measurement cases of the colouring path
    if name == "q13":
        return Workload("q13", "coloring", [queens(13, 13)], [13], S=1000, steps=3000, lr=0.01, n_colors=13,
                        recipe="colouring, queen13-13 (169 nodes, 3328 edges, Table 13) with K=13; S=1000; "
                               "3000 steps; lr 0.01 (the paper's largest COLOR instance, P:447)")
    if name == "k8":
        return Workload("k8", "coloring", [random_regular(100_000, 20, 8)], [8], S=64, steps=3000, lr=0.01,
                        n_colors=8, recipe="colouring, random 20-regular N=100,000 (seed 8) with K=8; S=64; "
                                           "3000 steps; lr 0.01 (scale case of the K-ary kernel)")
    raise KeyError(name)
