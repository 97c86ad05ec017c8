"""GPU parity for NEXT-1 (clamp map, sensitive transition, Eq. 11 / P:248) and NEXT-2
(Langevin noise, Eq. 9 / 11) through the C ABI, against the fp32
contract oracle: p within the BASELINE.json bar (1e-4 after 50 steps) and, under the
shared arithmetic contract, bit-identical theta / m / v / p and statistics."""
import numpy as np
import pytest

import gen
import oracle
from test_gpu_parity import assert_state_equal, assert_stats_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_02135_b200 as Q
    return Q


def gpu(Q, g, problem, S, seed, S_total=None, offset=0, **hp):
    cfg = Q.make_config(problem, S_total=S if S_total is None else S_total, seed=seed, replica_offset=offset,
                        S_local=S, **hp)
    return Q.Solver(g.rowptr, g.colidx, cfg)


def ocfg(problem, S, seed, threads=8, **hp):
    return oracle.make_cfg(problem, S=S, seed=seed, threads=threads, **hp)


CASES = [
    # (problem, graph, S, gamma_min, map, temperature, extra hyper-parameters)
    ("mis", lambda: gen.random_regular(256, 3, 1), 16, -2.0, "clamp", 0.0, {}),
    ("mis", lambda: gen.erdos_renyi(700, 0.15, 2000), 100, -2.0, "clamp", 0.0, dict(lr=0.3)),
    ("maxcut", lambda: gen.random_regular(2000, 5, 3), 64, -20.0, "clamp", 0.0, {}),
    ("maxclique", lambda: gen.erdos_renyi(120, 0.6, 6), 24, -2.0, "clamp", 0.0, dict(comm=0.5)),
    ("mis", lambda: gen.erdos_renyi(1500, 0.05, 4), 512, -2.0, "clamp", 0.001, dict(alpha=4)),
    ("mis", lambda: gen.random_regular(256, 3, 1), 16, -2.0, "sigmoid", 0.001, {}),
    ("maxcut", lambda: gen.erdos_renyi(500, 0.02, 9), 13, -5.0, "sigmoid", 0.01, dict(comm=1.0)),
    ("maxcut", lambda: gen.random_regular(3000, 5, 8), 200, -5.0, "clamp", 0.001, {}),
    ("mis", lambda: gen.erdos_renyi(400, 0.01, 8), 1, -2.0, "clamp", 0.001, {}),
    ("mis", lambda: gen.erdos_renyi(300, 0.2, 10), 1000, -2.0, "clamp", 0.001, dict(lr=0.1)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fifty_steps_parity(Q, case):
    problem, mk, S, gmin, mp, T, hp = CASES[case]
    g = mk()
    gam = oracle.schedule(gmin, 0.1, 1000)[:50]
    sol = gpu(Q, g, problem, S, 11, map=mp, temperature=T, **hp)
    st0 = oracle.init(g, ocfg(problem, S, 11, map=mp, temperature=T, **hp))
    assert_state_equal(sol, st0)                      # init (clamp: p_0 = 1/2 + U)
    sol.run(gam)
    st = oracle.run(g, ocfg(problem, S, 11, map=mp, temperature=T, **hp), gam)
    gs = assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    if mp == "clamp":
        assert np.array_equal(gs["theta"], gs["p"]) and gs["p"].min() >= 0 and gs["p"].max() <= 1


@pytest.mark.parametrize("mp,T", [("clamp", 0.0), ("clamp", 0.001), ("sigmoid", 0.001)])
def test_full_schedule_c1_with_evaluation(Q, mp, T):
    """All 1000 steps of c1 under the NEXT settings, then rounding (p >= 1/2 for clamp) and evaluation."""
    w = gen.workload("c1")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    hp.update(map=mp, temperature=T)
    sol = gpu(Q, g, "mis", w.S, w.seeds[0], **hp)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps)
    st = oracle.run(g, ocfg("mis", w.S, w.seeds[0], **hp), oracle.schedule(w.gamma_min, w.gamma_max, w.steps))
    assert_state_equal(sol, st)
    counts, energy, best = oracle.evaluate(g, "mis", 2.0, st.theta, map=mp)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
    assert res.best_replica == best and res.best_energy == energy[best]
    assert np.array_equal(res.best_x, (st.theta[:, best] >= oracle.threshold(mp)).astype(np.uint8))


def test_config_c3_clamp_noise_full_size(Q):
    """c3 (Max-Cut, 5-regular N=1e4, S=256) at full size under clamp + noise, 50 steps."""
    w = gen.workload("c3")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    hp.update(map="clamp", temperature=0.001)
    sol = gpu(Q, g, "maxcut", w.S, w.seeds[0], **hp)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 50)
    st = oracle.run(g, ocfg("maxcut", w.S, w.seeds[0], threads=16, **hp),
                    oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50])
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)


@pytest.mark.parametrize("mp", ["sigmoid", "clamp"])
def test_noise_keyed_by_global_replica(Q, mp):
    """With alpha_c = 0 the replicas are independent, so a shard [offset, offset+S_l) of S_total
    must reproduce exactly those columns of the full run: xi is keyed by the global replica."""
    g = gen.random_regular(500, 6, 2)
    gam = oracle.schedule(-2.0, 0.1, 200)[:40]
    full = gpu(Q, g, "mis", 96, 3, comm=0.0, map=mp, temperature=0.01)
    full.run(gam)
    fs = full.get_state()
    for off, S in [(0, 32), (32, 32), (40, 8), (88, 8), (33, 13), (61, 35)]:   # odd offsets split noise pairs
        sh = gpu(Q, g, "mis", S, 3, S_total=96, offset=off, comm=0.0, map=mp, temperature=0.01)
        sh.run(gam)
        ss = sh.get_state()
        for k in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[k], fs[k][:, off:off + S]), (off, k)


@pytest.mark.parametrize("SB", [8, 16])
def test_blocked_layout_clamp_noise(Q, monkeypatch, SB):
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", str(SB))
    g = gen.erdos_renyi(900, 0.02, 31)
    gam = oracle.schedule(-2.0, 0.1, 300)[:50]
    sol = gpu(Q, g, "mis", 100, 21, comm=0.3, map="clamp", temperature=0.001)
    sol.run(gam)
    st = oracle.run(g, ocfg("mis", 100, 21, comm=0.3, map="clamp", temperature=0.001), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)


def test_clamp_checkpoint_resume(Q):
    g = gen.erdos_renyi(500, 0.02, 3)
    gam = oracle.schedule(-2.0, 0.1, 100)
    a = gpu(Q, g, "mis", 40, 9, map="clamp", temperature=0.001)
    a.run(gam[:20])
    ck, cs = a.get_state(), a.get_stats()
    a.run(gam[20:40])
    b = gpu(Q, g, "mis", 40, 9, map="clamp", temperature=0.001)
    b.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=cs["c"])
    assert np.array_equal(b.get_state()["p"], ck["p"])
    b.run(gam[20:40])
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k])


def test_clamp_nonfinite_detected(Q):
    """Clamp would hide an inf / NaN (it maps them into [0, 1]): the flag is raised on the
    pre-map value. 1 - lr wd overflows to +inf, so p (1 - lr wd) is inf (or NaN at p = 0)."""
    g = gen.random_regular(50, 4, 1)
    sol = gpu(Q, g, "mis", 8, 1, lr=10.0, weight_decay=-1e38, map="clamp")
    sol.run_linear(-2.0, 0.1, 10)
    with pytest.raises(Q.QQAError) as e:
        sol.round_evaluate()
    assert e.value.status == 5


def test_invalid_map_and_temperature_rejected(Q):
    g = gen.random_regular(50, 4, 1)
    for bad in (dict(map=2), dict(temperature=-1.0), dict(temperature=float("nan"))):
        with pytest.raises(Q.QQAError) as e:
            gpu(Q, g, "mis", 8, 1, **bad)
        assert e.value.status == 1
