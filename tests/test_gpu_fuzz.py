"""Seeded random sweep of the option space through the C ABI against the fp32 contract oracle:
problem x map x noise x alpha x alpha_c x S (ragged) x graph family x replica blocking x batch x
schedule length (persistent vs launch-per-step, schedule-table chunks). Every case must be
bit-identical (theta, m, v, p, statistics) with integer evaluation equal."""
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


def _case(k):
    r = np.random.default_rng(1000 + k)
    problem = ["mis", "maxcut", "maxclique"][int(r.integers(3))]
    fam = int(r.integers(3))
    n = int(r.integers(20, 400)) if problem != "maxclique" else int(r.integers(10, 90))
    if problem == "maxclique":
        g = gen.erdos_renyi(n, float(r.uniform(0.3, 0.8)), 7 + k)
    elif fam == 0:
        g = gen.erdos_renyi(n, float(r.uniform(0.005, 0.1)), 7 + k)
    elif fam == 1:
        d = int(r.integers(1, 8))
        g = gen.random_regular(n - (n * d) % 2, d, 7 + k)
    else:
        g = gen.grid(int(r.integers(2, 20)), int(r.integers(2, 20)))
    batch = problem != "maxclique" and r.random() < 0.25
    gor = None
    if batch:
        parts = [g] + [gen.erdos_renyi(int(r.integers(5, 60)), 0.1, 50 + k + j) for j in range(int(r.integers(1, 4)))]
        g, gor = gen.disjoint_union(parts)
    S = int(r.choice([1, 2, 5, 8, 13, 31, 64, 100, 257]))
    hp = dict(alpha=int(r.choice([2, 4])), comm=float(r.choice([0.0, 0.1, 0.7])),
              map=str(r.choice(["sigmoid", "clamp"])), temperature=float(r.choice([0.0, 0.0, 0.003])),
              lr=float(r.choice([1.0, 0.3])))
    steps = int(r.choice([1, 2, 37, 120]))
    sb = str(r.choice(["", "", "8", "16"]))
    gmin = -5.0 if problem == "maxcut" else -2.0
    return problem, g, gor, S, hp, steps, sb, gmin


N_FUZZ = int(__import__("os").environ.get("QQA_FUZZ_CASES", "24"))
N_FUZZ_K = int(__import__("os").environ.get("QQA_FUZZ_CASES_K", "8"))


@pytest.mark.parametrize("k", range(N_FUZZ))
def test_random_configuration(Q, monkeypatch, k):
    problem, g, gor, S, hp, steps, sb, gmin = _case(k)
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    gam = oracle.schedule(gmin, 0.1, max(steps, 2) * 3)[:steps]
    cfg = Q.make_config(problem, S_total=S, seed=k + 3, **hp)
    sol = Q.Solver(g.rowptr, g.colidx, cfg, group_of_row=gor)
    sol.run(gam)
    csr = oracle.complement_groups(g, gor) if (problem == "maxclique" and gor is not None) else None
    st = oracle.run(g, oracle.make_cfg(problem, S=S, seed=k + 3, threads=8, **hp), gam, csr=csr)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    if gor is None:
        counts, energy, best = oracle.evaluate(g, problem, 2.0, st.theta, map=hp["map"])
        res = sol.round_evaluate()
        pr = res.per_replica
        assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
        assert res.best_replica == best
    else:
        G = int(gor.max()) + 1
        counts, energy, best = oracle.evaluate_groups(g, problem, 2.0, st.theta, gor, G, map=hp["map"])
        res = sol.round_evaluate_groups()
        assert np.array_equal(res.counts, counts) and np.array_equal(res.best_replica, best)


@pytest.mark.parametrize("k", range(N_FUZZ_K))
def test_random_colouring_configuration(Q, k):
    r = np.random.default_rng(5000 + k)
    K = int(r.integers(2, 17))
    g = [gen.queens(int(r.integers(3, 7)), int(r.integers(3, 7))), gen.mycielski(int(r.integers(2, 5))),
         gen.erdos_renyi(int(r.integers(10, 200)), 0.05, k)][int(r.integers(3))]
    S = int(r.choice([1, 3, 16, 33, 100]))
    hp = dict(alpha=int(r.choice([2, 4])), comm=float(r.choice([0.0, 0.2])), lr=float(r.choice([0.1, 0.03])),
              temperature=float(r.choice([0.0, 0.002])))
    steps = int(r.choice([1, 20, 60]))
    gam = oracle.schedule(-2.0, 0.1, 200)[:steps]
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=S, seed=k, n_colors=K, **hp))
    sol.run(gam)
    st = oracle.run_K(g, oracle.make_cfg("mis", S=S, seed=k, threads=8, **hp), K, gam)
    gs = sol.get_state()
    for f, ref in (("p", st.P), ("m", st.m), ("v", st.v)):
        assert np.array_equal(gs[f].view(np.uint32), ref.view(np.uint32)), f
    counts, energy, best, X = oracle.evaluate_K(g, st.P)
    res = sol.round_evaluate()
    assert np.array_equal(res.per_replica["violations"], counts[:, 1]) and res.best_replica == best
