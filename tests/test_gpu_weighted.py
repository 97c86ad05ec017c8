"""GPU parity for weighted graphs (MIS and Max-Cut, Optsicom-like +-1 weights):
bit-identical state against the fp32 contract oracle, exact weight sums in the evaluation, unit
weights equal to the unweighted path, and the graph checks on weights."""
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


def solver(Q, g, problem, S, seed, **hp):
    return Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=seed, **hp), weights=g.weights)


CASES = [("maxcut", "pm1", 64, -5.0, {}), ("maxcut", "uniform", 13, -5.0, dict(map="clamp", temperature=0.001)),
         ("mis", "int", 100, -2.0, dict(comm=0.3)), ("mis", "uniform", 256, -2.0, dict(alpha=4)),
         ("maxcut", "int", 8, -20.0, {})]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fifty_steps_parity_and_evaluation(Q, case):
    problem, kind, S, gmin, hp = CASES[case]
    g = gen.with_weights(gen.erdos_renyi(600, 0.02, 20 + case), kind, case)
    gam = oracle.schedule(gmin, 0.1, 1000)[:50]
    sol = solver(Q, g, problem, S, 7, **hp)
    sol.run(gam)
    st = oracle.run(g, oracle.make_cfg(problem, S=S, seed=7, threads=8, **hp), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    counts, energy, best, ws = oracle.evaluate(g, problem, 2.0, st.theta, map=hp.get("map", "sigmoid"), wsums=True)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
    assert np.array_equal(pr["wviolations"], ws[:, 0] * 2.0 ** -24) and np.array_equal(pr["wcut"], ws[:, 1] * 2.0 ** -24)
    assert np.array_equal(pr["energy"], energy) and res.best_replica == best


def test_full_schedule_weighted_maxcut(Q):
    g = gen.with_weights(gen.random_regular(3000, 6, 4), "pm1", 9)
    sol = solver(Q, g, "maxcut", 64, 3)
    sol.run_linear(-5.0, 0.1, 1000)
    st = oracle.run(g, oracle.make_cfg("maxcut", S=64, seed=3, threads=16), oracle.schedule(-5.0, 0.1, 1000))
    assert_state_equal(sol, st)
    _, energy, best = oracle.evaluate(g, "maxcut", 2.0, st.theta)
    res = sol.round_evaluate()
    assert res.best_replica == best and res.best_energy == energy[best]


def test_unit_weights_equal_unweighted(Q):
    g = gen.erdos_renyi(500, 0.03, 5)
    ones = np.ones(g.nnz, np.float32)
    for problem in ("mis", "maxcut"):
        a = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=24, seed=2))
        b = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=24, seed=2), weights=ones)
        for s in (a, b):
            s.run_linear(-2.0, 0.1, 200)
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(a.get_state()[f], b.get_state()[f]), (problem, f)
        ra, rb = a.round_evaluate(), b.round_evaluate()
        assert np.array_equal(ra.per_replica["energy"], rb.per_replica["energy"])


@pytest.mark.parametrize("SB", [8, 16])
def test_weighted_blocked_layout(Q, monkeypatch, SB):
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", str(SB))
    g = gen.with_weights(gen.erdos_renyi(800, 0.02, 31), "uniform", 3)
    gam = oracle.schedule(-5.0, 0.1, 300)[:40]
    sol = solver(Q, g, "maxcut", 100, 21, comm=0.3)
    sol.run(gam)
    st = oracle.run(g, oracle.make_cfg("maxcut", S=100, seed=21, comm=0.3), gam)
    assert_state_equal(sol, st)


def test_weight_checks(Q):
    g = gen.with_weights(gen.erdos_renyi(50, 0.2, 1), "pm1", 1)
    bad = g.weights.copy()
    bad[0] = 3.0                                           # w_ij != w_ji
    with pytest.raises(Q.QQAError) as e:
        Q.Solver(g.rowptr, g.colidx, Q.make_config("maxcut", S_total=8), weights=bad)
    assert e.value.status == 2
    bad[0] = np.nan
    with pytest.raises(Q.QQAError):
        Q.Solver(g.rowptr, g.colidx, Q.make_config("maxcut", S_total=8), weights=bad)
    for problem, extra in (("maxclique", {}), ("coloring", dict(n_colors=3)), ("maxclique_sparse", {})):
        with pytest.raises(Q.QQAError) as e:
            Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=8, **extra), weights=g.weights)
        assert e.value.status == 6
