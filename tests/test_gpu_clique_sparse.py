"""GPU parity for the printed max-clique relaxation on the original sparse graph (problem
"maxclique_sparse"): bit-identical state and statistics against the fp32 contract oracle,
complement counts equal to the dense-complement path, and a graph far beyond the dense limit."""
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


CASES = [(lambda: gen.erdos_renyi(120, 0.6, 6), 24, {}),
         (lambda: gen.erdos_renyi(300, 0.3, 7), 100, dict(comm=0.5, alpha=4)),
         (lambda: gen.random_regular(1000, 30, 8), 13, dict(map="clamp", temperature=0.001)),
         (lambda: gen.erdos_renyi(80, 0.7, 9), 1, {}),
         (lambda: gen.erdos_renyi(200, 0.5, 10), 257, dict(map="clamp"))]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fifty_steps_parity(Q, case):
    mk, S, hp = CASES[case]
    g = mk()
    gam = oracle.schedule(-2.0, 0.1, 1000)[:50]
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique_sparse", S_total=S, seed=11, **hp))
    sol.run(gam)
    st = oracle.run(g, oracle.make_cfg("maxclique_sparse", S=S, seed=11, threads=8, **hp), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    mp = hp.get("map", "sigmoid")
    counts, energy, best = oracle.evaluate(g, "maxclique_sparse", 2.0, st.theta, map=mp)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
    assert np.array_equal(pr["energy"], energy) and res.best_replica == best


def test_full_schedule_finds_a_clique_and_matches_dense_evaluation(Q):
    g = gen.erdos_renyi(150, 0.6, 12)
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique_sparse", S_total=64, seed=3))
    sol.run_linear(-2.0, 0.1, 2000)
    st = oracle.run(g, oracle.make_cfg("maxclique_sparse", S=64, seed=3, threads=8), oracle.schedule(-2.0, 0.1, 2000))
    assert_state_equal(sol, st)
    res = sol.round_evaluate()
    assert res.per_replica["violations"][res.best_replica] == 0          # a clique
    # the dense-complement handle evaluates the same theta identically
    dense = Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique", S_total=64, seed=3))
    s = sol.get_state()
    dense.set_state(s["theta"], s["m"], s["v"], s["step"])
    rd = dense.round_evaluate()
    for f in ("size", "violations", "cut", "energy"):
        assert np.array_equal(rd.per_replica[f], res.per_replica[f]), f
    assert rd.best_replica == res.best_replica and np.array_equal(rd.best_x, res.best_x)


@pytest.mark.parametrize("SB", [8, 16])
def test_blocked_layout(Q, monkeypatch, SB):
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", str(SB))
    g = gen.erdos_renyi(200, 0.4, 13)
    gam = oracle.schedule(-2.0, 0.1, 300)[:40]
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique_sparse", S_total=100, seed=5, comm=0.3))
    sol.run(gam)
    st = oracle.run(g, oracle.make_cfg("maxclique_sparse", S=100, seed=5, comm=0.3), gam)
    assert_state_equal(sol, st)


def test_beyond_the_dense_limit_sampled_rows(Q):
    """N = 200,000 (the dense complement path refuses n > 65,536): GPU step == oracle step on sampled rows."""
    g = gen.random_regular(200_000, 10, 14)
    with pytest.raises(Q.QQAError):
        Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique", S_total=16, seed=1))
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("maxclique_sparse", S_total=16, seed=1))
    cfg = oracle.make_cfg("maxclique_sparse", S=16, seed=1)
    gam = oracle.schedule(-2.0, 0.1, 100)
    rows = np.sort(np.random.default_rng(0).choice(g.n, 3000, replace=False)).astype(np.int32)
    sol.run(gam[:3])
    before, bstats = sol.get_state(), sol.get_stats()
    sol.run(gam[3:4])
    after, astats = sol.get_state(), sol.get_stats()
    out = oracle.step_rows(g, cfg, float(gam[3]), 4, before["p"], bstats["c"], bstats["sumD"], bstats["sumD2"],
                           before["theta"][rows], before["m"][rows], before["v"][rows], rows)
    for f in ("theta", "m", "v", "p"):
        assert np.array_equal(out[f].view(np.uint32), after[f][rows].view(np.uint32)), f
    assert np.array_equal(out["sumD"], astats["sumD"][rows])
