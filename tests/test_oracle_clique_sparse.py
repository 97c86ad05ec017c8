"""Pins for the printed max-clique relaxation on the original graph (problem "maxclique_sparse",
P:715; SURVEY.md §8(f) NEXT-3 option for large sparse graphs; reading R14). CPU only.

  l(p) = -1^T p + (lam/2) (1^T p (1^T p - 1) - p^T A p),  dl/dp_i = -1 + lam ((T - 1/2) - (A p)_i)

Pins: exactness at binary points against the MIS energy on the complement (exhaustive), the
closed-form interior identity printed = MIS-on-complement - (lam/8) s_{alpha=2} (reading R14),
central finite differences, the contract's fixed-point column sums, contract vs fp64, evaluation
identical to the dense-complement path, brute-force optimal cliques."""
import itertools

import numpy as np
import pytest

import gen
import oracle
from oracle import definition as D


def test_binary_points_equal_mis_on_complement_exhaustive():
    g = gen.erdos_renyi(9, 0.5, 21)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    Ac = D.complement_adjacency(A)
    X = np.array(list(itertools.product([0, 1], repeat=g.n)), float).T
    printed = D.relaxed_objective("maxclique_sparse", A, X)
    assert np.allclose(printed, D.relaxed_objective("mis", Ac, X))
    assert np.allclose(printed[:40], [D.printed_clique_energy(A, X[:, k]) for k in range(40)])


@pytest.mark.parametrize("lam", [2.0, 0.7])
def test_interior_identity_reading_R14(lam):
    """printed(p) = MIS_on_complement(p) - (lam/8) s_{alpha=2}(p) for every p in [0,1]^N."""
    g = gen.erdos_renyi(15, 0.4, 4)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P = np.random.default_rng(0).random((15, 9))
    lhs = D.relaxed_objective("maxclique_sparse", A, P, lam)
    rhs = D.relaxed_objective("mis", D.complement_adjacency(A), P, lam) - lam / 8.0 * D.entropy(P, 2)
    assert np.allclose(lhs, rhs, atol=1e-12)


@pytest.mark.parametrize("alpha,comm", [(2, 0.0), (4, 0.3)])
def test_gradient_finite_differences(alpha, comm):
    g = gen.erdos_renyi(9, 0.4, 5)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P = np.random.default_rng(2).uniform(0.05, 0.95, (9, 5))
    G = D.grad_p("maxclique_sparse", A, P, -1.1, alpha, 2.0, comm)
    h = 1e-6
    for i, s in itertools.product(range(9), range(5)):
        Pp, Pm = P.copy(), P.copy()
        Pp[i, s] += h
        Pm[i, s] -= h
        fd = (D.R_hat("maxclique_sparse", A, Pp, -1.1, alpha, 2.0, comm)
              - D.R_hat("maxclique_sparse", A, Pm, -1.1, alpha, 2.0, comm)) / (2 * h)
        assert abs(fd - G[i, s]) <= 1e-5 * max(1.0, abs(fd))


def test_contract_column_sums_are_exact_fixed_point():
    P = np.random.default_rng(3).random((5000, 7)).astype(np.float32)
    T = oracle.colsum(P)
    C = np.rint(P.astype(np.float64) * 2.0 ** 40).astype(np.int64).sum(axis=0)
    assert np.array_equal(T, (C.astype(np.float64) * 2.0 ** -40).astype(np.float32))
    assert np.allclose(T, P.astype(np.float64).sum(axis=0), rtol=1e-6)


def test_contract_matches_definition_one_and_fifty_steps():
    g = gen.erdos_renyi(50, 0.3, 8)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    cfg = oracle.make_cfg("maxclique_sparse", S=12, seed=5, comm=0.3)
    gam = oracle.schedule(-2.0, 0.1, 200)
    st = oracle.run(g, cfg, gam[:9])
    th1, m1, _ = D.run("maxclique_sparse", A, st.theta.astype(np.float64), [float(gam[9])], comm=float(np.float32(0.3)),
                       m0=st.m.astype(np.float64), v0=st.v.astype(np.float64), t0=st.t)
    oracle.run(g, cfg, gam[9:10], state=st)
    assert np.allclose(st.m, m1, rtol=1e-4, atol=1e-6) and np.allclose(st.theta, th1, rtol=1e-5, atol=1e-5)
    st50 = oracle.run(g, oracle.make_cfg("maxclique_sparse", S=12, seed=5), gam[:50])
    th, _, _ = D.run("maxclique_sparse", A, D.init_theta(g.n, 12, 5), gam[:50].astype(np.float64))
    assert np.abs(st50.p - D.sigmoid(th)).max() < 1e-4


def test_evaluation_equals_dense_complement_path():
    g = gen.erdos_renyi(60, 0.3, 9)
    theta = np.random.default_rng(4).normal(size=(60, 33)).astype(np.float32)
    theta[::7, ::5] = 0.0
    a = oracle.evaluate(g, "maxclique_sparse", 2.0, theta)
    b = oracle.evaluate(g, "maxclique", 2.0, theta)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    assert np.array_equal(a[0], D.counts("maxclique_sparse", A, D.round_x(theta)))


def test_bruteforce_max_clique():
    """Best of S=100 after 3000 steps is a maximum clique on >= 90% of ER(12, 0.5) instances."""
    hits, n_inst = 0, 25
    for k in range(n_inst):
        g = gen.erdos_renyi(12, 0.5, 6000 + k)
        opt, _ = D.brute_force("maxclique", D.dense_adjacency(g.n, g.rowptr, g.colidx))
        st = oracle.run(g, oracle.make_cfg("maxclique_sparse", S=100, seed=k + 1), oracle.schedule(-2.0, 0.1, 3000))
        counts, energy, best = oracle.evaluate(g, "maxclique_sparse", 2.0, st.theta)
        hits += energy[best] == opt
        assert counts[best, 1] == 0          # a clique: no non-adjacent pair inside
    assert hits >= 0.9 * n_inst
