"""Pins for weighted graphs ("for a weighted graph we simply let A_ij denote the edge weight";
the Optsicom Max-Cut family has weights in {-1, 0, 1}). CPU only.

Pins: unit weights reproduce the unweighted contract bit for bit (fl(1 p) = p), central finite
differences of the weighted relaxed objective, the weighted Max-Cut / MIS optimum by brute force,
exact fixed-point weight sums in the evaluation against the dense definition, contract vs fp64."""
import itertools

import numpy as np
import pytest

import gen
import oracle
from oracle import definition as D


def test_unit_weights_equal_unweighted_bit_for_bit():
    g = gen.erdos_renyi(200, 0.05, 3)
    gw = gen.Graph(g.n, g.rowptr, g.colidx, np.ones(g.nnz, np.float32))
    for problem in ("mis", "maxcut"):
        gam = oracle.schedule(-2.0, 0.1, 100)[:40]
        a = oracle.run(g, oracle.make_cfg(problem, S=12, seed=4), gam)
        b = oracle.run(gw, oracle.make_cfg(problem, S=12, seed=4), gam)
        for f in ("theta", "m", "v", "p", "sumD", "sumD2"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (problem, f)


@pytest.mark.parametrize("problem", ["mis", "maxcut"])
@pytest.mark.parametrize("kind", ["pm1", "uniform"])
def test_weighted_gradient_finite_differences(problem, kind):
    g = gen.with_weights(gen.erdos_renyi(9, 0.4, 5), kind, 6)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx, g.weights)
    P = np.random.default_rng(1).uniform(0.05, 0.95, (9, 4))
    G = D.grad_p(problem, A, P, -0.7, 2, 2.0, 0.0)
    h = 1e-6
    for i, s in itertools.product(range(9), range(4)):
        Pp, Pm = P.copy(), P.copy()
        Pp[i, s] += h
        Pm[i, s] -= h
        fd = (D.R_hat(problem, A, Pp, -0.7, 2, 2.0, 0.0) - D.R_hat(problem, A, Pm, -0.7, 2, 2.0, 0.0)) / (2 * h)
        assert abs(fd - G[i, s]) <= 1e-5 * max(1.0, abs(fd))


def test_evaluation_weight_sums_exact():
    g = gen.with_weights(gen.erdos_renyi(40, 0.3, 7), "int", 8)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx, g.weights)
    theta = np.random.default_rng(2).normal(size=(40, 21)).astype(np.float32)
    for problem in ("mis", "maxcut"):
        counts, energy, best, ws = oracle.evaluate(g, problem, 2.0, theta, wsums=True)
        X = D.round_x(theta)
        want = D.weighted_sums(A, X)
        assert np.array_equal(ws.astype(np.float64) * 2.0 ** -24, want)
        e = -want[:, 1] if problem == "maxcut" else -X.sum(axis=0) + 2.0 * want[:, 0]
        assert np.array_equal(energy, e) and best == D.best_replica(e)


def test_weighted_maxcut_bruteforce_pm1():
    """Weights in {-1, +1} (Optsicom-like): best of S=100 after 2000 steps hits the exhaustive optimum on
    >= 90% of ER(12, 0.4) instances."""
    hits, n_inst = 0, 20
    for k in range(n_inst):
        g = gen.with_weights(gen.erdos_renyi(12, 0.4, 300 + k), "pm1", k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx, g.weights)
        opt, _ = D.brute_force("maxcut", A)
        st = oracle.run(g, oracle.make_cfg("maxcut", S=100, seed=k + 1), oracle.schedule(-5.0, 0.1, 2000))
        _, energy, best = oracle.evaluate(g, "maxcut", 2.0, st.theta)
        hits += abs(energy[best] - opt) < 1e-9
    assert hits >= 0.9 * n_inst


def test_weighted_contract_matches_definition():
    g = gen.with_weights(gen.erdos_renyi(60, 0.1, 9), "uniform", 10)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx, g.weights)
    for problem in ("mis", "maxcut"):
        gam = oracle.schedule(-2.0, 0.1, 100)[:20]
        st = oracle.run(g, oracle.make_cfg(problem, S=8, seed=3), gam)
        th, _, _ = D.run(problem, A, D.init_theta(g.n, 8, 3), gam.astype(np.float64))
        assert np.abs(st.p - D.sigmoid(th)).max() < 1e-4
