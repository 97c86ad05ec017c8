"""Pins for the NEXT-1 / NEXT-2 parts of the oracle (CPU only):

  NEXT-1  sensitive transition with Clamp (Eq. 11; Clamp P:248): AdamW on p
          itself with dR/dp, then p <- Clamp(p'); rounding x = Theta(p - 1/2).
  NEXT-2  Langevin noise sqrt(2 eta T) xi (Eq. 9 / 11; T = 0.001 at P:670),
          xi from a counter-based Box-Muller generator (both sides implement it).

Each pin is something other than the oracle itself: closed forms (Adam's first step,
Theorem 1's gamma < 0 limit, the variance of a pure-noise random walk), libm / numpy
for the contract's own ln and cos, the normal distribution (scipy KS test), and brute
force on tiny graphs.
"""
import math

import numpy as np
import pytest
from scipy import stats

import gen
import oracle
from oracle import definition as D


# ------------------------------------------------------------- noise primitives
def test_contract_ln_within_three_ulp_of_libm():
    # every binade of (0, 1] the generator can produce (u1 >= 2^-24), dense near 1
    us = np.concatenate([np.float32(2.0) ** -np.arange(0, 25, dtype=np.float32),
                         np.linspace(2 ** -24, 1.0, 200001, dtype=np.float32),
                         np.float32(1.0) - np.arange(1, 2000, dtype=np.float32) * np.float32(2 ** -24)])
    for u in us[::5]:
        got, true = oracle.ln(float(u)), math.log(float(u))
        ulp = float(np.spacing(np.float32(abs(true)))) if true != 0 else 0.0
        assert abs(got - true) <= 3.0 * ulp + 1e-45, (u, got, true)


def test_contract_cos2pi_matches_libm():
    xs = np.arange(0, 1 << 24, 97, dtype=np.int64).astype(np.float64) * 2.0 ** -24
    got = np.array([oracle.cos2pi(float(x)) for x in xs[::50]])
    want = np.cos(2 * np.pi * xs[::50])
    assert np.abs(got - want).max() <= 3e-7
    assert oracle.cos2pi(0.0) == 1.0 and oracle.cos2pi(0.5) == -1.0
    assert oracle.cos2pi(0.25) == 0.0 and oracle.cos2pi(0.75) == 0.0


def test_contract_sin2pi_matches_libm():
    xs = np.arange(0, 1 << 24, 97, dtype=np.int64).astype(np.float64) * 2.0 ** -24
    got = np.array([oracle.sin2pi(float(x)) for x in xs[::50]])
    assert np.abs(got - np.sin(2 * np.pi * xs[::50])).max() <= 3e-7
    assert oracle.sin2pi(0.0) == 0.0 and oracle.sin2pi(0.25) == 1.0 and oracle.sin2pi(0.75) == -1.0


def test_paired_noise_halves_are_independent():
    """Replicas (2j, 2j+1) share one hash (cos / sin halves of Box-Muller): each half is N(0,1) and the
    two are uncorrelated (reading R24)."""
    z = D.gauss_noise(5, 3, 4000, 64)
    even, odd = z[:, 0::2].ravel(), z[:, 1::2].ravel()
    for h in (even, odd):
        assert stats.kstest(h, "norm").statistic < 3e-3
    assert abs(np.corrcoef(even, odd)[0, 1]) < 0.01
    assert abs(np.corrcoef(even ** 2, odd ** 2)[0, 1]) < 0.02   # not just uncorrelated: independent radii mix


def test_contract_noise_equals_fp64_box_muller():
    """Same integer hash -> the fp32 contract's xi is the fp64 Box-Muller value to rounding."""
    for seed, t, n, S in [(7, 1, 300, 64), (123456789, 2999, 50, 100), (0, 5, 1, 1)]:
        z32 = oracle.noise(seed, t, n, S).astype(np.float64)
        z64 = D.gauss_noise(seed, t, n, S)
        assert np.all(np.abs(z32 - z64) <= 2e-6 * (1.0 + np.abs(z64)))


def test_noise_is_standard_normal_and_independent():
    z = D.gauss_noise(11, 1, 2000, 256).ravel()
    assert abs(z.mean()) < 5 * 1.0 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / z.size)
    assert stats.kstest(z, "norm").statistic < 2e-3
    # different steps, variables, replicas and seeds are uncorrelated
    a, b = D.gauss_noise(11, 1, 1000, 64), D.gauss_noise(11, 2, 1000, 64)
    c = D.gauss_noise(12, 1, 1000, 64)
    for x, y in [(a, b), (a, c), (a[:, :-1], a[:, 1:]), (a[:-1], a[1:])]:
        assert abs(np.corrcoef(x.ravel(), y.ravel())[0, 1]) < 0.02
    zc = oracle.noise(11, 1, 2000, 256).ravel()
    assert stats.kstest(zc, "norm").statistic < 2e-3


# ---------------------------------------------------------------- clamp map
def test_clamp_init_is_half_plus_uniform():
    g = gen.random_regular(64, 3, 1)
    st = oracle.init(g, oracle.make_cfg("mis", S=24, seed=99, map="clamp"))
    want = D.init_p_clamp(g.n, 24, 99).astype(np.float32)
    assert np.array_equal(st.theta, want) and np.array_equal(st.p, want)
    assert (np.abs(st.p - 0.5) <= 0.01 + 1e-7).all()
    assert (st.c == 0.5).all()


def test_clamp01_special_values():
    assert oracle.clamp01(-3.0) == 0.0 and oracle.clamp01(7.0) == 1.0 and oracle.clamp01(0.25) == 0.25
    assert math.copysign(1.0, oracle.clamp01(-0.0)) == 1.0       # -0 -> +0
    assert oracle.clamp01(float("nan")) == 0.0


@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
def test_clamp_first_step_closed_form(problem):
    """Adam from m = v = 0: p_1 = Clamp(p_0 (1 - lr wd) - lr g / (|g| + eps)), g = dR/dp (no chain factor)."""
    g = gen.erdos_renyi(40, 0.2, 3) if problem != "maxclique" else gen.erdos_renyi(30, 0.7, 3)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    p0 = D.init_p_clamp(g.n, 10, 5).astype(np.float32).astype(np.float64)
    lr, wd, gam = 0.3, 0.01, -1.5
    grad = D.grad_p(problem, A, p0, gam, 2, 2.0, 0.2)
    want = np.clip(p0 * (1 - lr * wd) - lr * grad / (np.abs(grad) + 1e-8), 0.0, 1.0)
    got, _, _ = D.run(problem, A, p0, [gam], alpha=2, comm=0.2, lr=lr, wd=wd, map="clamp")
    assert np.allclose(got, want, atol=1e-12)
    cfg = oracle.make_cfg(problem, S=10, seed=5, map="clamp", lr=lr, comm=0.2)
    st = oracle.run(g, cfg, np.float32([gam]))
    assert np.abs(st.p - want).max() < 2e-6


def test_clamp_gamma_negative_limit_is_half():
    """Theorem 1, gamma < 0 with f = 0 (edgeless Max-Cut), no comm, no decay:
    p -> 1/2, the unique minimiser of gamma * s(p), under the clamp map too."""
    g = gen.edgeless(40)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    p0 = np.clip(0.5 + np.random.default_rng(1).uniform(-0.4, 0.4, (40, 8)), 0, 1)
    p, _, _ = D.run("maxcut", A, p0, [-2.0] * 3000, comm=0.0, lr=0.01, wd=0.0, map="clamp")
    assert np.abs(p - 0.5).max() < 1e-2
    st = oracle.run(g, oracle.make_cfg("maxcut", S=8, seed=2, map="clamp", lr=0.01, weight_decay=0.0, comm=0.0),
                    np.full(3000, -2.0, np.float32))
    assert np.abs(st.p - 0.5).max() < 1e-2


def test_clamp_stays_in_unit_box_and_ends_binary():
    """Clamp keeps p in [0, 1] at every step; gamma annealed to > 0 leaves p almost binary."""
    w = gen.workload("c1")
    g = w.graphs[0]
    cfg = oracle.make_cfg("mis", S=16, seed=1, map="clamp")
    gam = oracle.schedule(-2.0, 0.1, 1000)
    st = oracle.init(g, cfg)
    for k in range(0, 1000, 100):
        oracle.run(g, cfg, gam[k:k + 100], state=st)
        assert (st.p >= 0).all() and (st.p <= 1).all()
    assert np.mean((st.p == 0) | (st.p == 1)) > 0.95


@pytest.mark.parametrize("problem,alpha,comm", [("mis", 2, 0.1), ("maxcut", 4, 0.3), ("maxclique", 2, 0.0)])
def test_clamp_one_step_contract_matches_definition(problem, alpha, comm):
    g = gen.erdos_renyi(60, 0.12, 21) if problem != "maxclique" else gen.erdos_renyi(40, 0.7, 21)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    cfg = oracle.make_cfg(problem, S=12, seed=5, alpha=alpha, comm=comm, map="clamp", lr=0.3)
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 100)
    st = oracle.run(g, cfg, gam[:9])
    p1, m1, _ = D.run(problem, A, st.theta.astype(np.float64), [float(gam[9])], alpha=alpha, comm=comm,
                      lr=float(np.float32(0.3)), m0=st.m.astype(np.float64), v0=st.v.astype(np.float64),
                      t0=st.t, map="clamp")
    oracle.run(g, cfg, gam[9:10], state=st)
    assert np.allclose(st.m, m1, rtol=1e-4, atol=1e-6)
    assert np.allclose(st.p, p1, rtol=1e-5, atol=1e-5)
    assert np.array_equal(st.theta, st.p)


@pytest.mark.parametrize("mp,T,problem", [("clamp", 0.0, "mis"), ("clamp", 0.001, "mis"),
                                          ("sigmoid", 0.001, "mis"), ("clamp", 0.001, "maxcut")])
def test_fifty_steps_contract_matches_definition(mp, T, problem):
    """50 fp32 contract steps vs fp64 (BASELINE.json bar 1e-4 on p), NEXT-1 / NEXT-2 settings."""
    g = gen.workload("c1").graphs[0] if problem == "mis" else gen.random_regular(500, 5, 3)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    gmin = -2.0 if problem == "mis" else -5.0
    cfg = oracle.make_cfg(problem, S=16, seed=1, map=mp, temperature=T)
    gam = oracle.schedule(gmin, 0.1, 1000)[:50]
    st = oracle.run(g, cfg, gam)
    x0 = D.init_p_clamp(g.n, 16, 1) if mp == "clamp" else D.init_theta(g.n, 16, 1)
    th, _, _ = D.run(problem, A, x0.astype(np.float32).astype(np.float64), gam.astype(np.float64), map=mp,
                     temperature=float(np.float32(T)), seed=1)
    p = th if mp == "clamp" else D.sigmoid(th)
    assert np.abs(st.p - p).max() < 1e-4


@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
def test_clamp_bruteforce_optimum_on_small_er(problem):
    """The paper's own setting (Clamp): best of S=100 after 3000 steps hits the brute-force
    optimum on >= 90% of ER(12, 0.3) instances; MIS / clique best replicas are feasible."""
    hits, n_inst = 0, 25
    for k in range(n_inst):
        g = gen.erdos_renyi(12, 0.3, 5000 + k)
        A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
        opt, _ = D.brute_force(problem, A)
        cfg = oracle.make_cfg(problem, S=100, seed=k + 1, map="clamp", lr=0.3)
        st = oracle.run(g, cfg, oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 3000))
        counts, energy, best = oracle.evaluate(g, problem, 2.0, st.theta, map="clamp")
        hits += energy[best] == opt
        if problem != "maxcut":
            assert counts[best, 1] == 0
    assert hits >= 0.9 * n_inst


def test_clamp_eval_threshold_is_half():
    g = gen.erdos_renyi(30, 0.3, 4)
    A = D.dense_adjacency(g.n, g.rowptr, g.colidx)
    P = np.random.default_rng(0).random((30, 9)).astype(np.float32)
    P[:3] = 0.5                                              # Theta(0) = 1 at p = 1/2
    counts, energy, best = oracle.evaluate(g, "mis", 2.0, P, map="clamp")
    want = D.counts("mis", A, D.round_x(P, "clamp"))
    assert np.array_equal(counts, want) and (D.round_x(P, "clamp")[:3] == 1).all()


# ------------------------------------------------------------ Langevin noise
@pytest.mark.parametrize("mp", ["sigmoid", "clamp"])
def test_pure_noise_random_walk_variance(mp):
    """Zero gradient (edgeless Max-Cut, gamma = 0, alpha_c = 0, wd = 0): Adam's step is exactly 0,
    so after K steps w_K - w_0 = sqrt(2 lr T) sum_k xi_k with variance 2 lr T K (Eq. 9)."""
    n, S, K, lr, T = 400, 64, 10, 1.0, 0.001
    g = gen.edgeless(n)
    cfg = oracle.make_cfg("maxcut", S=S, seed=4, map=mp, temperature=T, lr=lr, weight_decay=0.0, comm=0.0,
                          init_lo=0.0, init_hi=0.0)
    st0 = oracle.init(g, cfg)
    st = oracle.run(g, cfg, np.zeros(K, np.float32), state=st0.copy())
    d = (st.theta - st0.theta).astype(np.float64).ravel()
    var = 2 * lr * T * K
    assert abs(d.mean()) < 5 * math.sqrt(var / d.size)
    assert abs(d.var() / var - 1.0) < 5 * math.sqrt(2.0 / d.size)
    # and it is exactly the contract's own sum of draws (no other term moved w)
    ns = oracle.noise_scale(cfg)
    assert ns == np.float32(math.sqrt(2 * lr * T))
    w = st0.theta.copy()
    for t in range(1, K + 1):   # the contract adds the draw with one fused multiply-add: fma(ns, xi, w)
        xi = oracle.noise(4, t, n, S)
        w = np.array([_fma32(np.float32(ns), x, y) for x, y in zip(xi.ravel(), w.ravel())],
                     np.float32).reshape(w.shape)
        if mp == "clamp":
            w = np.clip(w, 0, 1)
    assert np.array_equal(w, st.theta)


def _fma32(a, b, c) -> np.float32:
    """a * b + c rounded once to fp32 (round half to even), from exact rational arithmetic."""
    from fractions import Fraction
    x = Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c))
    if x == 0:
        return np.float32(0.0)
    sign, x = (-1, -x) if x < 0 else (1, x)
    e = x.numerator.bit_length() - x.denominator.bit_length()          # 2^e <= x < 2^(e+2)
    if x < Fraction(2) ** e:
        e -= 1
    m = x / Fraction(2) ** (e - 23)                                     # in [2^23, 2^24)
    q, r = divmod(m.numerator, m.denominator)
    if 2 * r > m.denominator or (2 * r == m.denominator and q % 2 == 1):
        q += 1
    return np.float32(sign * q * 2.0 ** (e - 23))


def test_temperature_zero_is_noise_free():
    g = gen.random_regular(100, 4, 2)
    gam = oracle.schedule(-2.0, 0.1, 30)
    a = oracle.run(g, oracle.make_cfg("mis", S=8, seed=3), gam)
    b = oracle.run(g, oracle.make_cfg("mis", S=8, seed=3, temperature=0.0), gam)
    c = oracle.run(g, oracle.make_cfg("mis", S=8, seed=3, temperature=1e-3), gam)
    assert np.array_equal(a.theta, b.theta) and not np.array_equal(a.theta, c.theta)


def test_clamp_nonfinite_aborts():
    g = gen.random_regular(20, 3, 1)
    with pytest.raises(FloatingPointError):
        oracle.run(g, oracle.make_cfg("mis", S=4, seed=1, lr=float("inf"), map="clamp"),
                   oracle.schedule(-2.0, 0.1, 5))
