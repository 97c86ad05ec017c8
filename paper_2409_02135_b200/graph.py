"""Graph input for the solver: symmetric CSR from an undirected edge list, and edge-list / DIMACS files.

The C ABI (include/qqa.h) takes a symmetric CSR with rows sorted, no self-loops and no duplicates,
and optional symmetric edge weights (A_ij is the edge weight). This module builds exactly
that from what users have: (u, v[, w]) edge lists, as arrays or files. Pure data preparation; every
step of the method runs in libqqa.so.
"""
from __future__ import annotations

import numpy as np


def csr_from_edges(n: int, u, v, w=None):
    """(rowptr int64 [n+1], colidx int32 [nnz], weights float32 [nnz] or None) of the undirected graph
    with edges (u_k, v_k). Self-loops are dropped; duplicate edges are merged (weights: the first one
    kept); both directions are stored; rows are sorted ascending."""
    u = np.asarray(u, np.int64).ravel()
    v = np.asarray(v, np.int64).ravel()
    if u.shape != v.shape:
        raise ValueError("u and v must have the same length")
    if u.size and (min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= n):
        raise ValueError("vertex index out of [0, n)")
    keep = u != v
    u, v = u[keep], v[keep]
    ww = None if w is None else np.asarray(w, np.float32).ravel()[keep]
    a, b = np.minimum(u, v), np.maximum(u, v)
    key = a * n + b
    key, first = np.unique(key, return_index=True)        # one record per undirected edge
    a, b = key // n, key % n
    rows = np.concatenate([a, b])
    cols = np.concatenate([b, a])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    weights = None
    if ww is not None:
        we = ww[first]
        weights = np.concatenate([we, we])[order].astype(np.float32)
    return rowptr, cols.astype(np.int32), weights


def read_edge_list(path: str, one_based: bool | None = None):
    """Read a graph file: DIMACS ("p edge N M" / "e u v" lines, 1-based) or a plain list of
    "u v [w]" lines ("#" / "%" / "c" comments). Returns (n, rowptr, colidx, weights or None).
    one_based: None = DIMACS files 1-based, plain lists 0-based."""
    us, vs, ws = [], [], []
    n_decl, dimacs = None, False
    with open(path) as f:
        for line in f:
            t = line.split()
            if not t or t[0][0] in "#%c":
                continue
            if t[0] == "p":
                n_decl, dimacs = int(t[2]), True
                continue
            if t[0] == "e":
                t = t[1:]
                dimacs = True
            us.append(int(t[0]))
            vs.append(int(t[1]))
            if len(t) > 2:
                ws.append(float(t[2]))
    base = (1 if dimacs else 0) if one_based is None else (1 if one_based else 0)
    u = np.asarray(us, np.int64) - base
    v = np.asarray(vs, np.int64) - base
    n = n_decl if n_decl is not None else (int(max(u.max(), v.max())) + 1 if u.size else 0)
    w = np.asarray(ws, np.float32) if ws and len(ws) == len(us) else None
    rowptr, colidx, weights = csr_from_edges(n, u, v, w)
    return n, rowptr, colidx, weights
