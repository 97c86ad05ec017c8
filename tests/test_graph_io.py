"""Product-side graph input (paper_2409_02135_b200.graph): CSR from edge lists and files must equal the
generator's canonical CSR, drop loops, merge duplicates and keep weights symmetric. CPU only."""
import numpy as np

import gen
from paper_2409_02135_b200 import csr_from_edges, read_edge_list


def test_matches_generator_csr():
    g = gen.erdos_renyi(300, 0.05, 3)
    u, v = g.edges()
    rp, ci, w = csr_from_edges(g.n, v, u)                 # reversed orientation on purpose
    assert np.array_equal(rp, g.rowptr) and np.array_equal(ci, g.colidx) and w is None


def test_loops_duplicates_and_weights():
    rp, ci, w = csr_from_edges(4, [0, 1, 1, 2, 3, 2], [1, 0, 1, 3, 2, 0], w=[5, 6, 7, 8, 9, 1])
    # edges {0,1} (weight 5, duplicate dropped), loop (1,1) dropped, {2,3} weight 8, {0,2} weight 1
    assert list(rp) == [0, 2, 3, 5, 6]
    assert list(ci) == [1, 2, 0, 0, 3, 2]
    assert list(w) == [5, 1, 5, 1, 8, 8]


def test_read_dimacs_and_plain(tmp_path):
    p = tmp_path / "g.col"
    p.write_text("c a comment\np edge 4 3\ne 1 2\ne 2 3\ne 4 1\n")
    n, rp, ci, w = read_edge_list(str(p))
    assert n == 4 and list(rp) == [0, 2, 4, 5, 6] and list(ci) == [1, 3, 0, 2, 1, 0] and w is None
    q = tmp_path / "g.txt"
    q.write_text("# u v w\n0 1 -1\n1 2 1\n")
    n, rp, ci, w = read_edge_list(str(q))
    assert n == 3 and list(ci) == [1, 0, 2, 1] and list(w) == [-1, -1, 1, 1]
    gw = gen.with_weights(gen.erdos_renyi(50, 0.2, 1), "pm1", 2)
    u, v = gw.edges()
    lines = []
    for a, b in zip(u, v):
        e = int(np.flatnonzero(gw.colidx[gw.rowptr[a]:gw.rowptr[a + 1]] == b)[0]) + gw.rowptr[a]
        lines.append(f"{a} {b} {gw.weights[e]:g}")
    r = tmp_path / "w.txt"
    r.write_text("\n".join(lines) + "\n")
    n, rp, ci, w = read_edge_list(str(r))
    assert np.array_equal(rp[:n + 1], gw.rowptr) and np.array_equal(ci, gw.colidx) and np.array_equal(w, gw.weights)
