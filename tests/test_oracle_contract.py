"""Pins for the fp32 contract oracle (oracle/contract.c) against the fp64
definition (itself pinned in test_oracle_definition.py), libm, closed forms,
networkx and brute force. CPU only."""
import math

import networkx as nx
import numpy as np
import pytest

import gen
import oracle
from oracle import definition as D


# --------------------------------------------------------------- sigmoid
def test_exp_neg_within_two_ulp_of_libm():
    a = np.linspace(0.0, 87.0, 100001).astype(np.float32)
    for x in a[::7]:
        got = oracle.exp_neg(float(x))
        true = math.exp(-float(x))
        ulp = float(np.spacing(np.float32(true)))
        assert abs(got - true) <= 2.0 * ulp, (x, got, true)


def test_sigmoid_accuracy_and_special_values():
    th = np.linspace(-100, 100, 200001).astype(np.float32)
    ps = oracle.sigmoid(th).astype(np.float64)
    pt = D.sigmoid(th.astype(np.float64))
    normal = (pt >= np.finfo(np.float32).tiny) & (np.abs(th) <= 87.0)  # contract cut-off |theta| > 87
    ulp = np.spacing(pt.astype(np.float32)).astype(np.float64)
    assert (np.abs(ps - pt)[normal] <= 2.5 * ulp[normal]).all()
    assert (np.abs(ps - pt)[~normal] <= 2e-38).all()       # subnormal range; |theta| > 87 -> exactly 0 or 1
    assert oracle.sigmoid(np.float32([0.0]))[0] == 0.5
    assert oracle.sigmoid(np.float32([200.0]))[0] == 1.0
    assert oracle.sigmoid(np.float32([-200.0]))[0] == 0.0
    # monotone non-decreasing
    assert (np.diff(ps) >= 0).all()


# ----------------------------------------------------------- scalars, stats
def test_schedule_matches_definition():
    for T in (1, 2, 3, 1000, 3000):
        got = oracle.schedule(-2.0, 0.1, T)
        want = D.gamma_schedule(float(np.float32(-2.0)), float(np.float32(0.1)), T).astype(np.float32)
        assert np.array_equal(got, want)


def test_step_scalars_match_formulae():
    cfg = oracle.make_cfg("mis", S=4, lr=0.7, weight_decay=0.01, alpha=4)
    for t in (1, 2, 10, 3000):
        k, a, s, r = oracle.step_scalars(cfg, t, -1.25)
        assert k == np.float32(-2 * 4 * -1.25)
        assert a == pytest.approx(1 - 0.7 * 0.01, rel=1e-7)
        b1, b2, lr = float(np.float32(0.9)), float(np.float32(0.999)), float(np.float32(0.7))
        assert s == pytest.approx(lr / (1 - b1 ** t), rel=1e-7)
        assert r == pytest.approx(1 / math.sqrt(1 - b2 ** t), rel=1e-7)


def test_fixed_point_stats_match_two_pass_std():
    rng = np.random.default_rng(0)
    cfg = oracle.make_cfg("mis", S=37, seed=3)
    for scale, center in [(0.0025, 0.5), (0.2, 0.5), (1e-3, 0.999), (0.5, 0.5)]:
        g = gen.edgeless(200)
        st = oracle.init(g, cfg)  # only to get shapes
        P = np.clip(rng.normal(center, scale, size=(200, 37)), 0, 1).astype(np.float32)
        c = np.float32(center)
        d = (P - c).astype(np.float32)
        sD = np.rint((d * np.float32(2.0 ** 40)).astype(np.float64)).astype(np.int64).sum(axis=1)
        dd = (d * d).astype(np.float32)
        sD2 = np.rint((dd * np.float32(2.0 ** 40)).astype(np.float64)).astype(np.int64).sum(axis=1)
        sd_true = D.std_rows(P.astype(np.float64))
        mu_true = P.astype(np.float64).mean(axis=1)
        for i in range(0, 200, 13):
            mu, sd = oracle.finalize(float(c), int(sD[i]), int(sD2[i]), 37)
            assert mu == pytest.approx(mu_true[i], abs=1e-7)
            assert sd == pytest.approx(sd_true[i], rel=2e-6, abs=2e-6)
        del st


# ------------------------------------------------------- init and dynamics
def test_init_matches_definition_hash():
    g = gen.random_regular(64, 3, 1)
    cfg = oracle.make_cfg("mis", S=24, seed=99)
    st = oracle.init(g, cfg)
    th = D.init_theta(g.n, 24, 99).astype(np.float32)
    assert np.array_equal(st.theta, th)
    assert np.array_equal(st.p, oracle.sigmoid(th))
    assert (st.c == 0.5).all() and (st.m == 0).all() and (st.v == 0).all()


def _state64(st):
    return st.theta.astype(np.float64), st.m.astype(np.float64), st.v.astype(np.float64)


@pytest.mark.parametrize("problem,gmin", [("mis", -2.0), ("maxcut", -20.0), ("maxclique", -2.0)])
@pytest.mark.parametrize("alpha", [2, 4])
def test_one_step_matches_definition(problem, gmin, alpha):
    """From the same (fp32) state, one contract step equals one fp64 step to fp32 rounding."""
    g = gen.erdos_renyi(60, 0.12, 21) if problem != "maxclique" else gen.erdos_renyi(40, 0.7, 21)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    cfg = oracle.make_cfg(problem, S=12, seed=5, alpha=alpha, comm=0.3)
    gam = oracle.schedule(gmin, 0.1, 100)
    st = oracle.run(g, cfg, gam[:7])           # a non-trivial interior state
    th, m, v = _state64(st)
    t = st.t + 1
    th1, m1, v1 = D.run(problem, A, th, [float(gam[7])], alpha=alpha, comm=0.3, m0=m, v0=v, t0=st.t)
    oracle.run(g, cfg, gam[7:8], state=st)
    # fp32-vs-fp64 rounding, amplified by Adam's m/sqrt(v) normalisation, stays ~1e-6;
    # a dropped or sign-flipped term moves theta by O(0.1).
    assert np.allclose(st.m, m1, rtol=1e-4, atol=1e-6)
    assert np.allclose(st.theta, th1, rtol=1e-5, atol=1e-5)
    assert t == st.t


def test_fifty_steps_mis_matches_definition_c1():
    """Config c1 (MIS, 3-regular N=256, S=16): fp32 contract vs fp64 after 50 steps, p within 1e-4."""
    w = gen.workload("c1")
    g = w.graphs[0]
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    cfg = oracle.make_cfg("mis", S=w.S, seed=w.seeds[0])
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50]
    st = oracle.run(g, cfg, gam)
    th, _, _ = D.run("mis", A, D.init_theta(g.n, w.S, w.seeds[0]), gam.astype(np.float64))
    assert np.abs(st.p - D.sigmoid(th)).max() < 1e-4


def test_fifty_steps_mis_matches_definition_20_regular():
    """The headline graph family (c5: MIS on a random 20-regular graph, S = 64, BASELINE.json configs[4]) at
    N = 2000: the fp32 contract against the fp64 definition (Eq. 6/7/10, App. D, AdamW P:220-222) after
    50 steps of c5's schedule, p within north_star's 1e-4 (survey Appendix E measured 5.2e-6)."""
    w = gen.workload("c5")
    g = gen.random_regular(2000, 20, 5)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    hp = {k: v for k, v in w.hparams().items() if k not in ("problem", "map", "temperature", "n_colors")}
    cfg = oracle.make_cfg("mis", S=w.S, seed=w.seeds[0], threads=4, **hp)
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50]
    st = oracle.run(g, cfg, gam)
    th, _, _ = D.run("mis", A, D.init_theta(g.n, w.S, w.seeds[0]), gam.astype(np.float64), alpha=w.alpha,
                     lam=w.penalty, comm=w.comm, lr=w.lr, wd=w.weight_decay)
    dp = np.abs(st.p - D.sigmoid(th)).max()
    assert dp < 1e-4, dp
    assert dp > 0.0   # two different arithmetics (fp32 contract vs fp64): the pin is not vacuous


def test_threads_bit_identical():
    g = gen.erdos_renyi(300, 0.05, 8)
    gam = oracle.schedule(-2.0, 0.1, 40)
    a = oracle.run(g, oracle.make_cfg("maxcut", S=20, seed=2, threads=1), gam)
    b = oracle.run(g, oracle.make_cfg("maxcut", S=20, seed=2, threads=4), gam)
    for f in ("theta", "m", "v", "p", "c", "sumD", "sumD2"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_step_rows_matches_full_step():
    g = gen.erdos_renyi(200, 0.05, 9)
    cfg = oracle.make_cfg("mis", S=8, seed=4)
    gam = oracle.schedule(-2.0, 0.1, 20)
    st = oracle.run(g, cfg, gam[:5])
    before = st.copy()
    oracle.run(g, cfg, gam[5:6], state=st)
    rows = np.array([0, 17, 199, 3], np.int32)
    out = oracle.step_rows(g, cfg, float(gam[5]), before.t + 1, before.p, before.c, before.sumD, before.sumD2,
                           before.theta[rows], before.m[rows], before.v[rows], rows)
    for f in ("theta", "m", "v", "p"):
        assert np.array_equal(out[f], getattr(st, f)[rows])
    for f in ("c", "sumD", "sumD2"):
        assert np.array_equal(out[f], getattr(st, f)[rows])


# ------------------------------------------------------------ evaluation
@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
def test_eval_counts_match_definition(problem):
    rng = np.random.default_rng(3)
    g = gen.erdos_renyi(40, 0.3, 77)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    theta = rng.normal(size=(g.n, 70)).astype(np.float32)
    theta[rng.random(theta.shape) < 0.05] = 0.0       # Theta(0) = 1 ties
    counts, energy, best = oracle.evaluate(g, problem, 2.0, theta)
    X = (theta >= 0).astype(np.int64)
    want = D.counts(problem, A, X)
    assert np.array_equal(counts, want)
    assert np.array_equal(energy, D.energy_from_counts(problem, want))
    assert best == D.best_replica(energy)


def test_complement_matches_dense():
    g = gen.erdos_renyi(30, 0.4, 5)
    rp, ci = oracle.complement(g)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    assert np.array_equal(D.dense_adjacency(g.n, rp, ci), D.complement_adjacency(A))


# ----------------------------------------------------------- whole method
def _solve(g, problem, S=100, steps=3000, seed=1, gmin=-2.0):
    cfg = oracle.make_cfg(problem, S=S, seed=seed)
    st = oracle.run(g, cfg, oracle.schedule(gmin, 0.1, steps))
    return oracle.evaluate(g, problem, 2.0, st.theta), st


@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
def test_bruteforce_optimum_on_small_er(problem):
    """SPEC.md:582 (AC-1): best of S=100 after 3000 steps hits the brute-force
    optimum on >= 90% of ER(12, 0.3) instances, and is always feasible for MIS."""
    hits, n_inst = 0, 25
    for k in range(n_inst):
        g = gen.erdos_renyi(12, 0.3, 5000 + k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        opt, _ = D.brute_force(problem, A)
        (counts, energy, best), _ = _solve(g, problem, seed=k + 1, gmin=-5.0 if problem == "maxcut" else -2.0)
        hits += energy[best] == opt
        if problem != "maxcut":
            assert counts[best, 1] == 0
    assert hits >= 0.9 * n_inst


def test_bipartite_maxcut_is_complete():
    """Bipartite graphs: best cut = |E| (SURVEY §8(c) pin)."""
    for g in (gen.cycle(40), gen.grid(6, 7), gen.random_bipartite(20, 25, 0.2, 3)):
        (counts, energy, best), _ = _solve(g, "maxcut", S=32, steps=1000, gmin=-5.0)
        assert counts[best, 2] == g.n_edges


def test_edgeless_mis_takes_everything():
    g = gen.edgeless(50)
    (counts, energy, best), st = _solve(g, "mis", S=8, steps=500)
    assert counts[best, 0] == 50 and counts[best, 1] == 0


def test_mis_feasible_and_near_networkx_on_larger_er():
    g = gen.erdos_renyi(60, 0.15, 42)
    (counts, energy, best), _ = _solve(g, "mis", S=64, steps=2000)
    G = nx.complement(nx.Graph(list(zip(*g.edges()))))
    G.add_nodes_from(range(g.n))
    _, opt = nx.max_weight_clique(G, weight=None)
    assert counts[best, 1] == 0
    assert counts[best, 0] >= opt - 1


def test_determinism():
    g = gen.erdos_renyi(100, 0.08, 1)
    (c1, e1, b1), s1 = _solve(g, "mis", S=10, steps=200)
    (c2, e2, b2), s2 = _solve(g, "mis", S=10, steps=200)
    assert np.array_equal(s1.theta, s2.theta) and np.array_equal(c1, c2) and b1 == b2


def test_nonfinite_aborts():
    g = gen.random_regular(20, 3, 1)
    cfg = oracle.make_cfg("mis", S=4, seed=1, lr=float("inf"))
    with pytest.raises(FloatingPointError):
        oracle.run(g, cfg, oracle.schedule(-2.0, 0.1, 5))
