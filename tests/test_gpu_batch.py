"""GPU parity for NEXT-3: a batch of instances annealed as one block-diagonal handle
 -- replica state bit-identical to the contract oracle on the union, and every
instance's integer counts / energies / best replica / x bit-exact against the oracle's
per-instance evaluation."""
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


def check_groups(res, U, gor, G, problem, theta, mp="sigmoid", S_total=None, off=0):
    counts, energy, best = oracle.evaluate_groups(U, problem, 2.0, theta, gor, G, map=mp)
    S_l = res.counts.shape[1]
    assert np.array_equal(res.counts, counts[:, off:off + S_l])
    assert np.array_equal(res.energy, energy[:, off:off + S_l])
    assert np.array_equal(res.best_replica, best)
    assert np.array_equal(res.best_energy, energy[np.arange(G), best])
    x = (theta >= oracle.threshold(mp)).astype(np.uint8)
    assert np.array_equal(res.best_x, x[np.arange(U.n), best[gor]])


def test_c2_all_instances_one_handle(Q):
    """c2 (16 x ER(N in [700, 800], 0.15), S=100) as ONE batched handle, 50 steps, full size."""
    w = gen.workload("c2")
    U, gor = w.batched()
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=w.S, seed=w.seeds[0], **hp), group_of_row=gor)
    assert sol.n_groups == 16
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 50)
    st = oracle.run(U, oracle.make_cfg("mis", S=w.S, seed=w.seeds[0], threads=16, **hp),
                    oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50])
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    check_groups(sol.round_evaluate_groups(), U, gor, 16, "mis", st.theta)
    # the ungrouped evaluation of a batch is the union's (counts summed over instances)
    cu, eu, bu = oracle.evaluate(U, "mis", 2.0, st.theta)
    res = sol.round_evaluate()
    assert np.array_equal(np.stack([res.per_replica["size"], res.per_replica["violations"],
                                    res.per_replica["cut"]], 1), cu)
    assert res.best_replica == bu


def test_t1_128_instances_one_handle(Q):
    """t1 (the paper's Table 1 batch: 128 x ER(N in [700, 800], 0.15), S = 100) as ONE batched handle at full size
    in bench.py's launch configuration (persistent kernel, non-FULL shape with pipelined index loads), 20 steps:
    state bit-exact on the union, every instance's counts / energies / best replica / x bit-exact."""
    w = gen.workload("t1")
    U, gor = w.batched()
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=w.S, seed=w.seeds[0], **hp), group_of_row=gor)
    assert sol.n_groups == 128 and sol.step_path() == "persistent"
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 20)
    st = oracle.run(U, oracle.make_cfg("mis", S=w.S, seed=w.seeds[0], threads=16, **hp),
                    oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:20])
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    check_groups(sol.round_evaluate_groups(), U, gor, 128, "mis", st.theta)


@pytest.mark.parametrize("problem,mp,T", [("maxcut", "clamp", 0.001), ("maxclique", "sigmoid", 0.0),
                                          ("mis", "clamp", 0.0)])
def test_batch_full_schedule(Q, problem, mp, T):
    if problem == "maxclique":
        gs = [gen.erdos_renyi(25 + 4 * k, 0.6, 40 + k) for k in range(5)]
    else:
        gs = [gen.erdos_renyi(60 + 13 * k, 0.1, 40 + k) for k in range(5)] + [gen.edgeless(7), gen.cycle(10)]
    U, gor = gen.disjoint_union(gs)
    G = len(gs)
    S, steps = 48, 400
    gmin = -5.0 if problem == "maxcut" else -2.0
    sol = Q.Solver(U.rowptr, U.colidx, Q.make_config(problem, S_total=S, seed=3, map=mp, temperature=T),
                   group_of_row=gor)
    sol.run_linear(gmin, 0.1, steps)
    csr = oracle.complement_groups(U, gor) if problem == "maxclique" else None
    st = oracle.run(U, oracle.make_cfg(problem, S=S, seed=3, threads=8, map=mp, temperature=T),
                    oracle.schedule(gmin, 0.1, steps), csr=csr)
    assert_state_equal(sol, st)
    check_groups(sol.round_evaluate_groups(), U, gor, G, problem, st.theta, mp)


def test_batch_shard_reports_its_columns(Q):
    """A replica shard (offset, S_local of S_total) reports its own columns; best is over its replicas
    only without a communicator (the NCCL all-gather makes it global)."""
    gs = [gen.erdos_renyi(50, 0.1, 70 + k) for k in range(3)]
    U, gor = gen.disjoint_union(gs)
    sol = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=64, seed=9, replica_offset=32, S_local=32,
                                                     comm=0.0), group_of_row=gor)
    sol.run_linear(-2.0, 0.1, 100)
    full = oracle.run(U, oracle.make_cfg("mis", S=64, seed=9, comm=0.0), oracle.schedule(-2.0, 0.1, 100))
    gs_ = sol.get_state()
    assert np.array_equal(gs_["theta"], full.theta[:, 32:])
    res = sol.round_evaluate_groups(want_x=False)
    counts, energy, _ = oracle.evaluate_groups(U, "mis", 2.0, full.theta, gor, 3)
    assert np.array_equal(res.counts, counts[:, 32:]) and np.array_equal(res.energy, energy[:, 32:])


@pytest.mark.parametrize("SB", [8, 32])
def test_batch_blocked_layout(Q, monkeypatch, SB):
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", str(SB))
    gs = [gen.erdos_renyi(200, 0.03, 90 + k) for k in range(4)]
    U, gor = gen.disjoint_union(gs)
    sol = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=100, seed=4, comm=0.3), group_of_row=gor)
    gam = oracle.schedule(-2.0, 0.1, 300)[:50]
    sol.run(gam)
    st = oracle.run(U, oracle.make_cfg("mis", S=100, seed=4, comm=0.3), gam)
    assert_state_equal(sol, st)
    check_groups(sol.round_evaluate_groups(), U, gor, 4, "mis", st.theta)


def test_batch_rejects_cross_instance_edges_and_bad_groups(Q):
    gs = [gen.random_regular(20, 3, 1), gen.random_regular(20, 3, 2)]
    U, gor = gen.disjoint_union(gs)
    cfg = Q.make_config("mis", S_total=8)
    bad = gor.copy()
    bad[5] = 1                                # row 5's edges now cross instances (and non-monotone)
    with pytest.raises(Q.QQAError) as e:
        Q.Solver(U.rowptr, U.colidx, cfg, group_of_row=bad)
    assert e.value.status == 2
    bad = gor.copy()
    bad[19], bad[20] = 1, 0                   # contiguous ranges required
    with pytest.raises(Q.QQAError):
        Q.Solver(U.rowptr, U.colidx, cfg, group_of_row=bad)
    with pytest.raises(Q.QQAError):
        Q.Solver(U.rowptr, U.colidx, cfg, group_of_row=gor, n_groups=1)   # group id out of range
    # a cross-instance edge with consistent groups: caught by the device validation
    u, v = U.edges()
    g2 = gen.from_edges(U.n, np.append(u, 3), np.append(v, 30))
    with pytest.raises(Q.QQAError) as e:
        Q.Solver(g2.rowptr, g2.colidx, cfg, group_of_row=gor)
    assert e.value.status == 2 and "instances" in str(e.value)


def test_single_group_matches_ungrouped(Q):
    g = gen.erdos_renyi(300, 0.05, 5)
    a = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=40, seed=2))
    b = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=40, seed=2), group_of_row=np.zeros(g.n, np.int32))
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 200)
    ra, rb = a.round_evaluate(), b.round_evaluate_groups()
    assert rb.best_replica[0] == ra.best_replica and rb.best_energy[0] == ra.best_energy
    assert np.array_equal(rb.best_x, ra.best_x)
    rc = a.round_evaluate_groups()          # ungrouped handle: one instance
    assert rc.best_replica[0] == ra.best_replica and np.array_equal(rc.energy[0], ra.per_replica["energy"])
