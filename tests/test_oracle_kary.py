"""Pins for the K-ary / graph-colouring oracle (NEXT-4; App. B, map P:672-676,
energy P:745-750). CPU only. Each pin is external to the oracle: the paper's Table 13
graph statistics, its Proposition (s_K = s at K = 2), the closed-form extremes of s_K,
exactness of the relaxation at one-hot points, central finite differences, Adam's
first-step closed form, the gamma < 0 limit (Theorem 1 analogue: P -> 1/K), brute-force
optimal colourings and chromatic facts (bipartite = 2-colourable, chi(myciel3) = 4)."""
import itertools

import numpy as np
import pytest

import gen
import oracle
from oracle import definition as D


def _graph(name):
    if name.startswith("queen"):
        r, c = name[5:].split("-")
        return gen.queens(int(r), int(c))
    return gen.mycielski(int(name[6:]))


def test_colour_graph_generators_match_table_13(golden):
    for name, row in golden("color_graphs.json")["graphs"].items():
        g = _graph(name)
        assert (g.n, g.n_edges) == (row["nodes"], row["edges"]), name


def test_mycielski_is_triangle_free():
    g = gen.mycielski(5)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    assert np.trace(A @ A @ A) == 0


# ---------------------------------------------------------------- entropy
def test_sK_equals_binary_alpha_entropy_at_K2():
    """Proposition: with p_i2 = 1 - p_i1, s_2 = s (Eq. 7)."""
    rng = np.random.default_rng(0)
    p = rng.random((30, 5))
    P = np.stack([p, 1 - p], axis=2)
    for alpha in (2, 4, 6):
        assert np.allclose(D.entropy_K(P, alpha), D.entropy(p, alpha), atol=1e-12)


@pytest.mark.parametrize("K", [2, 3, 5, 9])
@pytest.mark.parametrize("alpha", [2, 4])
def test_sK_extremes(K, alpha):
    """s_K = N at the simplex centre (max), 0 at every one-hot point (min), in between elsewhere."""
    N, S = 7, 3
    assert np.allclose(D.entropy_K(np.full((N, S, K), 1.0 / K), alpha), N)
    X = np.random.default_rng(K).integers(0, K, (N, S))
    assert np.allclose(D.entropy_K(np.eye(K)[X], alpha), 0.0, atol=1e-12)
    P = np.random.default_rng(1).dirichlet(np.ones(K), (N, S))
    e = D.entropy_K(P, alpha)
    assert (e > 0).all() and (e < N).all()


def test_coloring_relaxation_exact_at_one_hot():
    g = gen.erdos_renyi(20, 0.3, 3)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    X = np.random.default_rng(2).integers(0, 4, (20, 6))
    assert np.allclose(D.coloring_objective(A, np.eye(4)[X]), D.conflicts(A, X))
    # brute-force count over edge list
    u, v = g.edges()
    assert np.array_equal(D.conflicts(A, X), (X[u] == X[v]).sum(axis=0))


# --------------------------------------------------------------- gradient
@pytest.mark.parametrize("alpha,comm,gamma", [(2, 0.0, -1.3), (4, 0.0, 0.7), (2, 0.3, -2.0), (4, 0.5, 0.1)])
def test_grad_K_finite_differences(alpha, comm, gamma):
    g = gen.erdos_renyi(8, 0.4, 5)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P = np.random.default_rng(3).dirichlet(np.ones(3), (8, 5))
    G = D.grad_K(A, P, gamma, alpha, comm)
    h = 1e-6
    for idx in itertools.islice(itertools.product(range(8), range(5), range(3)), 0, None, 7):
        Pp, Pm = P.copy(), P.copy()
        Pp[idx] += h
        Pm[idx] -= h
        fd = (D.R_hat_K(A, Pp, gamma, alpha, comm) - D.R_hat_K(A, Pm, gamma, alpha, comm)) / (2 * h)
        assert abs(fd - G[idx]) <= 1e-5 * max(1.0, abs(fd)), (idx, fd, G[idx])


# ------------------------------------------------------------------- map
def test_clamp_normalize_properties():
    rng = np.random.default_rng(4)
    W = rng.normal(0.2, 0.5, (50, 7, 5))
    P = D.clamp_normalize(W)
    assert (P >= 0).all() and np.allclose(P.sum(axis=2), 1.0)
    assert np.allclose(D.clamp_normalize(P), P)                       # idempotent on the simplex
    W[0, 0] = -1.0                                                   # every clamp 0 -> uniform (reading)
    assert np.allclose(D.clamp_normalize(W)[0, 0], 1 / 5)
    w = np.float32([[-0.2, 0.3, 1.7, 0.1]])
    assert np.allclose(oracle.normalize_K(w[0]), np.clip(w[0], 0, 1) / np.clip(w[0], 0, 1).sum(), atol=1e-7)


@pytest.mark.parametrize("through_map", [True, False])
def test_first_step_closed_form_K(through_map):
    """Adam from m = v = 0: P_1 = normalise(P_0 (1 - lr wd) - lr g / (|g| + eps)), g the gradient
    through the map (R33) or dR/dP (R29)."""
    g = gen.queens(4, 4)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P0 = D.clamp_normalize(D.init_W_K(g.n, 6, 4, 9))
    lr, wd, gam = 0.1, 0.01, -1.0
    G = (D.grad_K_map if through_map else D.grad_K)(A, P0, gam, 2, 0.2)
    want = D.clamp_normalize(P0 * (1 - lr * wd) - lr * G / (np.abs(G) + 1e-8))
    got, _, _ = D.run_K(A, P0, [gam], alpha=2, comm=0.2, lr=lr, wd=wd, through_map=through_map)
    assert np.allclose(got, want, atol=1e-12)


@pytest.mark.parametrize("alpha,comm,gamma", [(2, 0.0, -1.0), (4, 0.3, 0.5)])
def test_grad_K_map_is_the_chain_rule_through_the_map(alpha, comm, gamma):
    """Reading R33 pinned by central finite differences: at W = P (on the simplex, inside the clamp
    range) dR/dW of R(clamp_normalize(W)) equals g - <g, P> per (variable, replica) row."""
    g = gen.queens(4, 4)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    rng = np.random.default_rng(3)
    P = rng.dirichlet(np.full(5, 4.0), (g.n, 3))            # interior points, rows sum to 1
    G = D.grad_K_map(A, P, gamma, alpha, comm)
    h = 1e-6
    for (i, s_, k) in [(0, 0, 0), (3, 1, 2), (7, 2, 4), (15, 0, 3)]:
        Wp, Wm = P.copy(), P.copy()
        Wp[i, s_, k] += h
        Wm[i, s_, k] -= h
        fd = (D.R_hat_K(A, D.clamp_normalize(Wp), gamma, alpha, comm)
              - D.R_hat_K(A, D.clamp_normalize(Wm), gamma, alpha, comm)) / (2 * h)
        assert abs(fd - G[i, s_, k]) <= 1e-5 * max(1.0, abs(fd)), (i, s_, k, fd, G[i, s_, k])


def test_gradient_through_the_map_reproduces_table_4_small_queens():
    """Evidence for R33 (Table 4): the gradient through the map colours queen6-6 with 7
    colours and queen7-7 with 7 without a conflict, where dR/dP (R29) leaves conflicts."""
    for (r, K) in [(6, 7), (7, 7)]:
        gq = gen.queens(r, r)
        st = oracle.run_K(gq, oracle.make_cfg("mis", S=64, seed=1, lr=0.1, threads=4, temperature=0.001), K,
                          oracle.schedule(-2.0, 0.1, 2000))
        _, energy, best, _ = oracle.evaluate_K(gq, st.P)
        assert energy[best] == 0


def test_gamma_negative_limit_is_simplex_centre():
    """Theorem 1 analogue for s_K: no edges, no comm, no decay, gamma < 0 -> P = 1/K."""
    g = gen.edgeless(30)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P0 = np.random.default_rng(5).dirichlet(np.ones(4), (30, 6))
    P, _, _ = D.run_K(A, P0, [-2.0] * 3000, comm=0.0, lr=0.01, wd=0.0)
    assert np.abs(P - 0.25).max() < 1e-2
    cfg = oracle.make_cfg("mis", S=6, seed=3, lr=0.01, weight_decay=0.0, comm=0.0, init_lo=-0.2, init_hi=0.2)
    st = oracle.run_K(g, cfg, 4, np.full(3000, -2.0, np.float32))
    assert np.abs(st.P - 0.25).max() < 1e-2


# -------------------------------------------------------- contract vs fp64
def test_contract_init_matches_definition():
    g = gen.queens(5, 5)
    st = oracle.init_K(g, oracle.make_cfg("mis", S=12, seed=8), 5)
    want = D.clamp_normalize(D.init_W_K(g.n, 12, 5, 8).astype(np.float32).astype(np.float64))
    assert np.abs(st.P - want).max() < 1e-7
    assert np.allclose(st.P.sum(axis=2), 1.0, atol=1e-6) and (st.c == np.float32(0.2)).all()


def test_contract_kt_matches_formula():
    for K, alpha, gam in [(2, 2, -2.0), (5, 4, 0.1), (13, 2, -0.7)]:
        cK = 1.0 / ((K - 1) * ((K - 1) ** (alpha - 1) + 1))
        assert oracle.kt_K(K, alpha, gam) == np.float32(-float(np.float32(gam)) * cK * alpha * K)


@pytest.mark.parametrize("K,T,comm", [(5, 0.0, 0.1), (3, 0.001, 0.3), (9, 0.001, 0.0)])
def test_ten_steps_contract_matches_definition(K, T, comm):
    """K-ary dynamics amplify rounding differences (like Max-Cut, survey Appendix E): fp32 vs fp64
    drifts to ~1e-4 by step 20-50, so the contract is pinned to fp64 over 10 steps, where a dropped
    or wrong term moves P by > 1e-3. (GPU parity is bitwise against the contract.)"""
    g = gen.queens(5, 5) if K == 5 else (gen.erdos_renyi(40, 0.2, 6) if K == 3 else gen.queens(8, 8))
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    S = 16
    cfg = oracle.make_cfg("mis", S=S, seed=1, lr=0.1, temperature=T, comm=comm)
    gam = oracle.schedule(-2.0, 0.1, 1000)[:10]
    st = oracle.run_K(g, cfg, K, gam)
    P0 = D.clamp_normalize(D.init_W_K(g.n, S, K, 1).astype(np.float32).astype(np.float64))
    P, _, _ = D.run_K(A, P0, gam.astype(np.float64), lr=float(np.float32(0.1)), comm=float(np.float32(comm)),
                      temperature=float(np.float32(T)), seed=1)
    assert np.abs(st.P - P).max() < 2e-5


def test_contract_eval_matches_definition():
    g = gen.erdos_renyi(30, 0.3, 4)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P = np.random.default_rng(6).dirichlet(np.ones(4), (30, 11)).astype(np.float32)
    P[0, 0] = [0.25, 0.25, 0.25, 0.25]                          # tie -> lowest colour
    counts, energy, best, X = oracle.evaluate_K(g, P)
    assert X[0, 0] == 0 and np.array_equal(X, D.round_K(P))
    conf = D.conflicts(A, D.round_K(P))
    assert np.array_equal(counts[:, 1], conf) and np.array_equal(counts[:, 2], g.n_edges - conf)
    assert best == D.best_replica(energy)


# ----------------------------------------------------------- whole method
def test_bruteforce_optimal_colourings():
    """Best of S=64 after 2000 steps reaches the brute-force minimum conflicts (K=3) on >= 90% of
    ER(9, 0.4) instances."""
    hits, n_inst = 0, 20
    for k in range(n_inst):
        g = gen.erdos_renyi(9, 0.4, 700 + k)
        opt = D.brute_force_coloring(D.dense_adjacency(g.n, g.rowptr, g.colidx), 3)
        st = oracle.run_K(g, oracle.make_cfg("mis", S=64, seed=k + 1, lr=0.1, threads=4), 3,
                          oracle.schedule(-2.0, 0.1, 2000))
        _, energy, best, _ = oracle.evaluate_K(g, st.P)
        hits += energy[best] == opt
    assert hits >= 0.9 * n_inst


@pytest.mark.parametrize("K,g", [(2, gen.grid(6, 7)), (2, gen.cycle(40)), (2, gen.random_bipartite(20, 25, 0.2, 3)),
                                 (4, gen.mycielski(3)), (5, gen.queens(5, 5))])
def test_proper_colourings_found(K, g):
    """Bipartite graphs with K = 2 (the K = 2 colouring cost is |E| - cut), myciel3 with chi = 4,
    queen5-5 with 5 colours (Table 4 reports 0 conflicts for PQQA): a conflict-free replica."""
    st = oracle.run_K(g, oracle.make_cfg("mis", S=100, seed=1, lr=0.1, threads=4), K,
                      oracle.schedule(-2.0, 0.1, 3000))
    _, energy, best, X = oracle.evaluate_K(g, st.P)
    assert energy[best] == 0


def test_pure_noise_walk_K():
    """Zero gradient and a centred start: P' = P + sqrt(2 lr T) xi exactly, then the K-ary map."""
    n, S, K = 50, 16, 3
    g = gen.edgeless(n)
    cfg = oracle.make_cfg("mis", S=S, seed=4, temperature=0.001, weight_decay=0.0, comm=0.0,
                          init_lo=0.0, init_hi=0.0)
    st0 = oracle.init_K(g, cfg, K)
    st = oracle.run_K(g, cfg, K, np.zeros(1, np.float32), state=st0.copy())      # gamma = 0: g = q = 0
    ns = np.float32(oracle.noise_scale(cfg))
    xi = D.gauss_noise_K(4, 1, n, S, K)
    w = (st0.P + ns * xi.astype(np.float32)).astype(np.float32)
    want = np.stack([oracle.normalize_K(w[i, s]) for i in range(n) for s in range(S)]).reshape(n, S, K)
    assert np.abs(st.P - want).max() < 2e-6


def test_nonfinite_aborts_K():
    g = gen.queens(4, 4)
    with pytest.raises(FloatingPointError):
        oracle.run_K(g, oracle.make_cfg("mis", S=4, seed=1, lr=10.0, weight_decay=-1e38), 4,
                     oracle.schedule(-2.0, 0.1, 5))
