"""Input generators (gen/): structure, statistics, determinism."""
import numpy as np
import pytest

import gen


def _check_csr(g):
    assert g.rowptr[0] == 0 and g.rowptr[-1] == len(g.colidx)
    assert (np.diff(g.rowptr) >= 0).all()
    for i in range(g.n):
        row = g.colidx[g.rowptr[i]:g.rowptr[i + 1]]
        assert (np.diff(row) > 0).all()          # sorted, no duplicates
        assert not (row == i).any()              # no self loops
        for j in row:                            # symmetric
            rj = g.colidx[g.rowptr[j]:g.rowptr[j + 1]]
            assert np.searchsorted(rj, i) < len(rj) and rj[np.searchsorted(rj, i)] == i


@pytest.mark.parametrize("n,d", [(256, 3), (1000, 20), (500, 100), (10, 9)])
def test_rrg_regular_and_simple(n, d):
    g = gen.random_regular(n, d, 5)
    assert (g.degrees() == d).all() and g.n_edges == n * d // 2
    if n <= 1000:
        _check_csr(g)


def test_rrg_rejects_odd():
    with pytest.raises(ValueError):
        gen.random_regular(5, 3, 1)


def test_er_edge_count_statistics():
    # mean |E| of G(100, 0.1) over many seeds ~ 495 +- 3 sigma/sqrt(k)
    counts = [gen.erdos_renyi(100, 0.1, s).n_edges for s in range(200)]
    sigma = np.sqrt(4950 * 0.1 * 0.9)
    assert abs(np.mean(counts) - 495) < 3 * sigma / np.sqrt(200)
    assert gen.erdos_renyi(10, 0.0, 1).n_edges == 0
    assert gen.erdos_renyi(10, 1.0, 1).n_edges == 45
    _check_csr(gen.erdos_renyi(80, 0.3, 2))


def test_deterministic():
    a, b = gen.random_regular(300, 4, 9), gen.random_regular(300, 4, 9)
    assert np.array_equal(a.colidx, b.colidx)
    c = gen.random_regular(300, 4, 10)
    assert not np.array_equal(a.colidx, c.colidx)
    assert np.array_equal(gen.erdos_renyi(200, 0.1, 3).colidx, gen.erdos_renyi(200, 0.1, 3).colidx)


def test_workload_shapes():
    assert gen.c2_sizes() == gen.c2_sizes() and all(700 <= n <= 800 for n in gen.c2_sizes())
    assert 9000 <= gen.c4_size() <= 11000
    w = gen.workload("c1")
    assert w.graphs[0].n == 256 and w.S == 16 and w.steps == 1000
    w = gen.workload("c3")
    assert w.problem == "maxcut" and (w.graphs[0].degrees() == 5).all()


def test_bipartite_helpers():
    for g in (gen.cycle(8), gen.grid(3, 5), gen.random_bipartite(6, 7, 0.4, 2)):
        _check_csr(g)
        # 2-colourable: BFS colouring has no monochromatic edge
        col = -np.ones(g.n, int)
        for s0 in range(g.n):
            if col[s0] >= 0:
                continue
            col[s0] = 0
            stack = [s0]
            while stack:
                u = stack.pop()
                for v in g.colidx[g.rowptr[u]:g.rowptr[u + 1]]:
                    if col[v] < 0:
                        col[v] = 1 - col[u]
                        stack.append(v)
                    assert col[v] != col[u]
