"""Pins for the fp64 definition oracle (oracle/definition.py) against things
other than itself: SPEC/PAPER worked values (tests/golden), central finite
differences, closed forms (Prop. A.2, Theorem 1 limits), networkx and brute force."""
import itertools

import networkx as nx
import numpy as np
import pytest

import gen
from oracle import definition as D


def adj(n, edges):
    A = np.zeros((n, n))
    for a, b in edges:
        A[a, b] = A[b, a] = 1.0
    return A


# ------------------------------------------------------- worked values
def test_mis_single_edge(golden):
    w = golden("worked_values.json")["mis_single_edge"]
    A = adj(w["n"], w["edges"])
    for c in w["cases"]:
        x = np.array(c["x"], float)[:, None]
        assert D.discrete_energy("mis", A, x, w["lam"])[0] == c["energy"]


def test_clique_energy_printed_and_as_mis_on_complement(golden):
    w = golden("worked_values.json")["clique_triangle_and_path"]
    for c in w["cases"]:
        A = adj(c["n"], c["edges"])
        x = np.array(c["x"], float)
        assert D.printed_clique_energy(A, x, w["lam"]) == c["energy"]
        assert D.discrete_energy("maxclique", A, x[:, None], w["lam"])[0] == c["energy"]


def test_maxcut_small(golden):
    w = golden("worked_values.json")["maxcut_small"]
    c0, c1 = w["cases"]
    A = adj(c0["n"], c0["edges"])
    assert D.discrete_energy("maxcut", A, np.array(c0["x"], float)[:, None])[0] == c0["energy"]
    A = adj(c1["n"], c1["edges"])
    best, _ = D.brute_force("maxcut", A)
    assert best == c1["optimum"]


def test_mis_grad_half(golden):
    w = golden("worked_values.json")["mis_grad_half"]
    A = adj(w["n"], w["edges"])
    g = D.grad_objective("mis", A, np.array(w["p"])[:, None], w["lam"])[:, 0]
    assert np.array_equal(g, np.array(w["grad"]))


def test_maxcut_relaxed_half(golden):
    w = golden("worked_values.json")["maxcut_relaxed_half"]
    g = gen.erdos_renyi(30, 0.2, 7)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    val = D.relaxed_objective("maxcut", A, np.full((g.n, 1), 0.5))[0]
    assert val == pytest.approx(w["factor"] * g.n_edges, abs=1e-12)


def test_entropy_alpha4(golden):
    w = golden("worked_values.json")["entropy_alpha4"]
    assert D.entropy(np.array([[w["p"]]]), w["alpha"])[0] == pytest.approx(w["value"], abs=1e-15)


def test_qqa_objective_single_edge(golden):
    w = golden("worked_values.json")["qqa_objective_single_edge"]
    A = adj(w["n"], w["edges"])
    P = np.array(w["p"])[:, None]
    r = D.relaxed_objective("mis", A, P, w["lam"])[0] + w["gamma"] * D.entropy(P, w["alpha"])[0]
    assert r == pytest.approx(w["value"], abs=1e-15)


def test_std_half_half(golden):
    w = golden("worked_values.json")["std_half_half"]
    assert D.std_rows(np.array([w["column"]], float))[0] == w["std"]


def test_adamw_one_step(golden):
    w = golden("worked_values.json")["adamw_one_step"]
    th, m, v = D.adamw_step(np.array([0.3]), np.zeros(1), np.zeros(1), np.array([w["g"]]), 1,
                            w["lr"], 0.9, 0.999, 1e-8, 0.0)
    assert th[0] - 0.3 == pytest.approx(w["delta"], abs=1e-8)


def test_adamw_one_step_closed_form_any_g():
    # from m = v = 0: theta_1 = theta_0 (1 - lr wd) - lr g / (|g| + eps)  (SURVEY §8(c) AdamW pin)
    rng = np.random.default_rng(0)
    g = rng.normal(size=50) * 10 ** rng.uniform(-3, 3, 50)
    th0 = rng.normal(size=50)
    th, _, _ = D.adamw_step(th0, np.zeros(50), np.zeros(50), g, 1, 0.7, 0.9, 0.999, 1e-8, 0.01)
    expect = th0 * (1 - 0.7 * 0.01) - 0.7 * g / (np.abs(g) + 1e-8)
    assert np.allclose(th, expect, rtol=1e-12, atol=1e-12)


def test_gamma_schedule(golden):
    w = golden("worked_values.json")["gamma_midpoint"]
    gs = D.gamma_schedule(w["gamma_min"], w["gamma_max"], 3)
    assert gs[0] == w["gamma_min"] and gs[-1] == pytest.approx(w["gamma_max"], abs=1e-15)
    assert gs[1] == pytest.approx(w["mid"], abs=1e-15)
    assert D.gamma_schedule(-2.0, 0.1, 1)[0] == -2.0


# ----------------------------------------------- exactness & symmetries
@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
def test_relaxation_exact_at_binary_points(problem):
    """l_hat(x) = l(x) for x in {0,1}^N, l(x) from integer edge counts."""
    rng = np.random.default_rng(1)
    for k in range(20):
        g = gen.erdos_renyi(10, 0.35, 100 + k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        X = rng.integers(0, 2, size=(g.n, 30))
        # independent count: loop over edges explicitly
        B = D.problem_adjacency(problem, A)
        for s in range(X.shape[1]):
            x = X[:, s]
            size = int(x.sum())
            pairs = [(i, j) for i in range(g.n) for j in range(i + 1, g.n) if B[i, j]]
            viol = sum(x[i] & x[j] for i, j in pairs)
            cut = sum(x[i] ^ x[j] for i, j in pairs)
            direct = -cut if problem == "maxcut" else -size + 2.0 * viol
            assert D.discrete_energy(problem, A, X[:, s:s + 1].astype(float))[0] == pytest.approx(direct)
        c = D.counts(problem, A, X)
        assert np.allclose(D.energy_from_counts(problem, c), D.discrete_energy(problem, A, X.astype(float)))


def test_maxcut_spin_symmetry():
    g = gen.erdos_renyi(12, 0.4, 3)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    X = np.random.default_rng(2).integers(0, 2, size=(g.n, 40)).astype(float)
    assert np.allclose(D.discrete_energy("maxcut", A, X), D.discrete_energy("maxcut", A, 1 - X))


def test_clique_duality_exhaustive():
    """printed clique energy on G == MIS energy on the complement, all x."""
    g = gen.erdos_renyi(8, 0.5, 11)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    Ac = D.complement_adjacency(A)
    for bits in itertools.product([0, 1], repeat=g.n):
        x = np.array(bits, float)
        assert D.printed_clique_energy(A, x) == pytest.approx(D.discrete_energy("mis", Ac, x[:, None])[0])


# ------------------------------------------------------ finite differences
@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
@pytest.mark.parametrize("alpha", [2, 4])
@pytest.mark.parametrize("comm", [0.0, 0.3])
def test_grad_p_matches_finite_differences(problem, alpha, comm):
    rng = np.random.default_rng(alpha * 10 + int(comm * 10))
    g = gen.erdos_renyi(9, 0.4, 5)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    S = 5
    P = rng.uniform(0.05, 0.95, size=(g.n, S))
    assert D.std_rows(P).min() > 1e-3
    gamma, lam = -0.7, 2.0
    G = D.grad_p(problem, A, P, gamma, alpha, lam, comm)
    h = 1e-5
    for i in range(g.n):
        for s in range(S):
            Pp, Pm = P.copy(), P.copy()
            Pp[i, s] += h
            Pm[i, s] -= h
            fd = (D.R_hat(problem, A, Pp, gamma, alpha, lam, comm) -
                  D.R_hat(problem, A, Pm, gamma, alpha, lam, comm)) / (2 * h)
            assert abs(fd - G[i, s]) <= 1e-5 * max(1.0, abs(fd)), (i, s, fd, G[i, s])


def test_grad_theta_chain_rule_fd():
    rng = np.random.default_rng(9)
    g = gen.erdos_renyi(8, 0.4, 6)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    th = rng.normal(size=(g.n, 4))
    G = D.grad_theta("maxcut", A, th, 0.3, 4, 2.0, 0.2)
    h = 1e-6
    for i, s in [(0, 0), (3, 2), (7, 3)]:
        tp, tm = th.copy(), th.copy()
        tp[i, s] += h
        tm[i, s] -= h
        fd = (D.R_hat("maxcut", A, D.sigmoid(tp), 0.3, 4, 2.0, 0.2) -
              D.R_hat("maxcut", A, D.sigmoid(tm), 0.3, 4, 2.0, 0.2)) / (2 * h)
        assert abs(fd - G[i, s]) <= 1e-5 * max(1.0, abs(fd))


def test_entropy_shape():
    """s = N at p=1/2 (max), 0 at binary points, and CONCAVE per coordinate (s'' <= 0).

    P:145 calls s 'convex'; its second derivative -4a(a-1)(2p-1)^(a-2) is <= 0, so
    it is concave and gamma*s is convex for gamma < 0 (reading R22)."""
    for alpha in (2, 4, 6):
        assert D.entropy(np.full((7, 1), 0.5), alpha)[0] == 7
        assert D.entropy(np.array([[0.0], [1.0], [1.0]]), alpha)[0] == 0
        h = 1e-4
        for p in np.linspace(0.01, 0.99, 99):
            s = [D.entropy(np.array([[p + d]]), alpha)[0] for d in (-h, 0.0, h)]
            assert (s[0] - 2 * s[1] + s[2]) / h ** 2 <= 1e-6


# ------------------------------------------------------------ Prop. A.2
def test_prop_a2_bruteforce(golden):
    for c in golden("prop_a2.json")["cases"]:
        S, N = c["S"], c["N"]
        target = c.get("max_var", c.get("max_var_num", 0) / c.get("max_var_den", 1))
        best, arg = -1.0, []
        for bits in itertools.product([0, 1], repeat=S * N):
            P = np.array(bits, float).reshape(N, S)
            val = D.std_rows(P).sum()
            if val > best + 1e-12:
                best, arg = val, [P]
            elif abs(val - best) <= 1e-12:
                arg.append(P)
        assert best == pytest.approx(N * np.sqrt(target), abs=1e-12)
        for P in arg:  # every maximiser has floor/ceil(S/2) ones in every column
            ones = P.sum(axis=1)
            assert set(ones.tolist()) <= {S // 2, (S + 1) // 2}
        # and a continuous interior point never beats it
        rng = np.random.default_rng(S)
        for _ in range(200):
            assert D.std_rows(rng.uniform(size=(N, S))).sum() <= best + 1e-12


def test_comm_identical_replicas_zero():
    P = np.tile(np.random.default_rng(0).uniform(size=(6, 1)), (1, 5))
    assert D.comm_term(P, 0.7) == 0.0
    assert np.all(D.grad_comm(P, 0.7) == 0.0)


# ------------------------------------------------------- Theorem 1 limits
def test_theorem1_negative_gamma_converges_to_half():
    """gamma < 0 fixed, f = 0 (edgeless Max-Cut), alpha_c = 0: minimiser p = 1/2."""
    n, S = 6, 4
    A = np.zeros((n, n))
    th0 = np.random.default_rng(3).uniform(-2, 2, size=(n, S))
    th, _, _ = D.run("maxcut", A, th0, np.full(3000, -1.0), alpha=2, comm=0.0, lr=0.05, wd=0.0)
    assert np.abs(D.sigmoid(th) - 0.5).max() < 1e-4


def test_theorem1_positive_gamma_drives_binary():
    """At the end of the -2 -> 0.1 schedule the mean entropy per node is <= 0.01."""
    g = gen.erdos_renyi(40, 0.15, 12)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    th0 = D.init_theta(g.n, 8, 12)
    th, _, _ = D.run("mis", A, th0, D.gamma_schedule(-2.0, 0.1, 1500))
    P = D.sigmoid(th)
    assert (D.entropy(P, 2) / g.n).max() <= 0.01


# --------------------------------------------------------- brute force
def test_bruteforce_mis_matches_networkx():
    for k in range(15):
        g = gen.erdos_renyi(11, 0.3, 300 + k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        best, arg = D.brute_force("mis", A)
        G = nx.complement(nx.from_numpy_array(A))
        clique, w = nx.max_weight_clique(G, weight=None)
        assert best == -w
        for x in arg:
            assert D.counts("mis", A, x[:, None])[0, 1] == 0


def test_bruteforce_clique_matches_networkx():
    for k in range(10):
        g = gen.erdos_renyi(11, 0.5, 400 + k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        best, _ = D.brute_force("maxclique", A)
        _, w = nx.max_weight_clique(nx.from_numpy_array(A), weight=None)
        assert best == -w


def test_bruteforce_maxcut_bipartite_cuts_everything():
    for g in (gen.cycle(10), gen.grid(3, 4), gen.random_bipartite(5, 6, 0.5, 1)):
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        best, _ = D.brute_force("maxcut", A)
        assert best == -g.n_edges


# ------------------------------------------------------------------ init
def test_init_theta_uniform_and_shard_invariant():
    th = D.init_theta(500, 64, 7)
    assert th.min() >= -0.01 and th.max() < 0.01
    assert abs(th.mean()) < 5e-4 and abs(th.std() - 0.02 / np.sqrt(12)) < 3e-4
    assert np.array_equal(th, D.init_theta(500, 64, 7))
    assert not np.array_equal(th, D.init_theta(500, 64, 8))
