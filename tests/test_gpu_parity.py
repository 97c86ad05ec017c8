"""GPU parity: the CUDA path (through the C ABI) against the fp32 contract oracle.

Bar (BASELINE.json north_star): replica state p within max-abs 1e-4 after 50
fp32 steps, integer evaluation bit-exact. The arithmetic contract
makes the expected result bit-identical, which is asserted as well.
"""
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

TOL_P = 1e-4  # BASELINE.json: "p matches to max-abs 1e-4 after 50 fp32 steps"


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


def assert_state_equal(sol, st, exact=True, cols=None):
    gs = sol.get_state()
    ref = {k: getattr(st, k) if cols is None else getattr(st, k)[:, cols] for k in ("theta", "m", "v", "p")}
    dp = np.abs(gs["p"].astype(np.float64) - ref["p"]).max() if ref["p"].size else 0.0
    assert dp <= TOL_P, f"max |p_gpu - p_oracle| = {dp}"
    if exact:
        for k in ("theta", "m", "v", "p"):
            bad = np.count_nonzero(gs[k].view(np.uint32) != ref[k].view(np.uint32))
            assert bad == 0, f"{k}: {bad} of {gs[k].size} elements differ bitwise (max |d|={np.abs(gs[k]-ref[k]).max()})"
    return gs


def assert_stats_equal(sol, st):
    s = sol.get_stats()
    assert np.array_equal(s["c"].view(np.uint32), st.c.view(np.uint32))
    assert np.array_equal(s["sumD"], st.sumD)
    assert np.array_equal(s["sumD2"], st.sumD2)


# ------------------------------------------------------------------ sigmoid
def test_sigmoid_bit_exact_audit(Q):
    """T9: GPU sigmoid (via set_state -> p) equals the contract bit for bit on a dense sweep."""
    n, S = 4096, 256
    th = np.linspace(-95.0, 95.0, n * S).astype(np.float32)
    rng = np.random.default_rng(0)
    th[: n * S // 2] = rng.normal(0, 8, n * S // 2).astype(np.float32)
    th = th.reshape(n, S)
    g = gen.edgeless(n)
    sol = gpu(Q, g, "mis", S, 1)
    sol.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    p = sol.get_state()["p"]
    ref = oracle.sigmoid(th)
    assert np.count_nonzero(p.view(np.uint32) != ref.view(np.uint32)) == 0


# --------------------------------------------------------------------- init
@pytest.mark.parametrize("S", [1, 3, 13, 16, 64, 100, 256, 512, 1000])
def test_init_parity(Q, S):
    g = gen.random_regular(300, 4, 2)
    sol = gpu(Q, g, "mis", S, 77)
    st = oracle.init(g, ocfg("mis", S, 77))
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)


def test_init_shard_is_a_column_slice(Q):
    g = gen.random_regular(200, 4, 3)
    st = oracle.init(g, ocfg("mis", 96, 5))
    for off, S in [(0, 32), (32, 32), (64, 32), (40, 8)]:
        sol = gpu(Q, g, "mis", S, 5, S_total=96, offset=off)
        gs = sol.get_state()
        assert np.array_equal(gs["theta"], st.theta[:, off:off + S])


# -------------------------------------------------------------- dynamics
CASES = [
    # (problem, graph builder, S, gamma_min, alpha, comm)
    ("mis", lambda: gen.random_regular(256, 3, 1), 16, -2.0, 2, 0.1),
    ("mis", lambda: gen.erdos_renyi(700, 0.15, 2000), 100, -2.0, 2, 0.1),
    ("maxcut", lambda: gen.random_regular(2000, 5, 3), 64, -20.0, 2, 0.1),
    ("maxcut", lambda: gen.erdos_renyi(500, 0.02, 9), 13, -2.0, 4, 1.0),
    ("mis", lambda: gen.erdos_renyi(1500, 0.05, 4), 512, -2.0, 4, 0.5),
    ("mis", lambda: gen.random_regular(3000, 20, 5), 8, -2.0, 2, 0.0),
    ("maxclique", lambda: gen.erdos_renyi(120, 0.6, 6), 24, -2.0, 2, 0.1),
    ("mis", lambda: gen.erdos_renyi(400, 0.01, 8), 1, -2.0, 2, 0.1),      # S=1: comm term vanishes
    ("mis", lambda: gen.erdos_renyi(300, 0.2, 10), 1000, -2.0, 2, 0.1),   # paper's S=1000
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fifty_steps_parity(Q, case):
    problem, mk, S, gmin, alpha, comm = CASES[case]
    g = mk()
    gam = oracle.schedule(gmin, 0.1, 1000)[:50]
    sol = gpu(Q, g, problem, S, 11, alpha=alpha, comm=comm)
    sol.run(gam)
    st = oracle.run(g, ocfg(problem, S, 11, alpha=alpha, comm=comm), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_fifty_steps_full_size(Q, name):
    """BASELINE.json configs at full size, 50 steps, launch configuration of bench.py."""
    w = gen.workload(name, n_instances=2 if name == "c2" else None)
    for g, seed in zip(w.graphs, w.seeds):
        gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50]
        sol = gpu(Q, g, w.problem, w.S, seed, **{k: v for k, v in w.hparams().items() if k != "problem"})
        sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 50)
        st = oracle.run(g, ocfg(w.problem, w.S, seed, threads=16,
                                **{k: v for k, v in w.hparams().items() if k != "problem"}), gam)
        assert_state_equal(sol, st)
        assert_stats_equal(sol, st)
        # evaluation of identical rounded solutions: bit-exact integers
        counts, energy, best = oracle.evaluate(g, w.problem, w.penalty, st.theta)
        res = sol.round_evaluate()
        pr = res.per_replica
        assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
        assert np.array_equal(pr["energy"], energy)
        assert res.best_replica == best and res.best_energy == energy[best]
        assert np.array_equal(res.best_x, (st.theta[:, best] >= 0).astype(np.uint8))


def test_c5_sampled_rows_full_size(Q):
    """c5 (MIS, 20-regular, N=1e6, S=64) at full size in bench.py's launch configuration:
    GPU state after k steps -> one oracle step on sampled rows == GPU step k+1."""
    w = gen.workload("c5")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = gpu(Q, g, "mis", w.S, w.seeds[0], **hp)
    st0 = oracle.init(gen.Graph(g.n, g.rowptr, g.colidx), ocfg("mis", w.S, w.seeds[0], threads=16, **hp))
    rows = np.sort(np.random.default_rng(0).choice(g.n, 4000, replace=False)).astype(np.int32)
    gs = sol.get_state()
    assert np.array_equal(gs["theta"][rows], st0.theta[rows]) and np.array_equal(gs["p"], st0.p)
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)
    cfg = ocfg("mis", w.S, w.seeds[0], **hp)
    for k in (0, 1, 2, 7):
        sol.run_linear(w.gamma_min, w.gamma_max, w.steps, sol.get_state()["step"], k)  # catch up to step k
        before, bstats = sol.get_state(), sol.get_stats()
        assert before["step"] == k
        sol.run_linear(w.gamma_min, w.gamma_max, w.steps, k, k + 1)
        after, astats = sol.get_state(), sol.get_stats()
        out = oracle.step_rows(g, cfg, float(gam[k]), k + 1, before["p"], bstats["c"], bstats["sumD"],
                               bstats["sumD2"], before["theta"][rows], before["m"][rows], before["v"][rows], rows)
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(out[f].view(np.uint32), after[f][rows].view(np.uint32)), (k, f)
        assert np.array_equal(out["sumD"], astats["sumD"][rows]) and np.array_equal(out["sumD2"], astats["sumD2"][rows])


def test_c5_fifty_steps_full_size_bitwise(Q):
    """The headline config (c5: MIS, 20-regular N=1e6, S=64, bench.py's launch configuration: replica blocks
    of 32, k_step<4,1,0,FULL>) at FULL size for 50 steps: every element of theta / m / v / p and the int64
    statistics bit-exact against the contract oracle (north_star: p within 1e-4 after 50 fp32 steps), then
    the rounded solutions' integer counts bit-exact against oracle.evaluate."""
    w = gen.workload("c5")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = gpu(Q, g, "mis", w.S, w.seeds[0], **hp)
    assert sol.replica_block() == 32 and sol.step_path() == "step"
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 50)
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:50]
    st = oracle.run(g, ocfg("mis", w.S, w.seeds[0], threads=os.cpu_count() or 8, **hp), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    counts, energy, best = oracle.evaluate(g, "mis", w.penalty, st.theta)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
    assert np.array_equal(pr["energy"], energy)
    assert res.best_replica == best and res.best_energy == energy[best]
    assert np.array_equal(res.best_x, (st.theta[:, best] >= 0).astype(np.uint8))


def test_20_regular_full_schedule_replica_blocks_of_32(Q, monkeypatch):
    """c5's graph family and kernel late in the anneal: MIS on a 20-regular graph (N = 2000, S = 64) with
    QQA_BLOCK_REPLICAS=32 -- the replica-blocked layout and k_step<4,1,0,FULL> that c5 runs -- over the
    whole 3000-step schedule of c5, bit-exact against the contract oracle, then evaluation bit-exact."""
    w = gen.workload("c5")
    g = gen.random_regular(2000, 20, 5)
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", "32")
    sol = gpu(Q, g, "mis", w.S, w.seeds[0], **hp)
    assert sol.replica_block() == 32 and sol.step_path() == "step"
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps)
    st = oracle.run(g, ocfg("mis", w.S, w.seeds[0], threads=os.cpu_count() or 8, **hp),
                    oracle.schedule(w.gamma_min, w.gamma_max, w.steps))
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    counts, energy, best = oracle.evaluate(g, "mis", w.penalty, st.theta)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(np.stack([pr["size"], pr["violations"], pr["cut"]], 1), counts)
    assert res.best_replica == best and res.best_energy == energy[best]
    assert pr["violations"][best] == 0


def test_full_schedule_c1_bit_exact(Q):
    """All 1000 steps of c1, then rounding / evaluation / best replica."""
    w = gen.workload("c1")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = gpu(Q, g, "mis", w.S, w.seeds[0], **hp)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps)
    st = oracle.run(g, ocfg("mis", w.S, w.seeds[0], **hp), oracle.schedule(w.gamma_min, w.gamma_max, w.steps))
    assert_state_equal(sol, st)
    counts, energy, best = oracle.evaluate(g, "mis", 2.0, st.theta)
    res = sol.round_evaluate()
    assert res.best_replica == best and res.best_energy == energy[best]
    assert res.per_replica["violations"][best] == 0     # MIS feasible


# ------------------------------------------------------------------ API
def test_run_linear_equals_run(Q):
    g = gen.erdos_renyi(400, 0.03, 2)
    a = gpu(Q, g, "maxcut", 32, 3)
    b = gpu(Q, g, "maxcut", 32, 3)
    a.run_linear(-5.0, 0.1, 200, 0, 30)
    b.run(oracle.schedule(-5.0, 0.1, 200)[:30])
    sa, sb = a.get_state(), b.get_state()
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(sa[k], sb[k])


def test_checkpoint_resume(Q):
    g = gen.erdos_renyi(500, 0.02, 3)
    gam = oracle.schedule(-2.0, 0.1, 100)
    a = gpu(Q, g, "mis", 40, 9)
    a.run(gam[:20])
    ck, cs = a.get_state(), a.get_stats()
    a.run(gam[20:40])
    b = gpu(Q, g, "mis", 40, 123)  # different seed: state comes from the checkpoint
    b.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=cs["c"])
    assert np.array_equal(b.get_stats()["sumD"], cs["sumD"])
    b.run(gam[20:40])
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k])


def test_reset_restarts_identically(Q):
    g = gen.random_regular(300, 6, 4)
    a = gpu(Q, g, "mis", 16, 4)
    s0 = a.get_state()
    a.run_linear(-2.0, 0.1, 50)
    a.reset()
    s1 = a.get_state()
    assert s1["step"] == 0 and np.array_equal(s0["theta"], s1["theta"]) and np.array_equal(s0["m"], s1["m"])


@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique", "maxclique_sparse", "coloring"])
@pytest.mark.parametrize("breakit", ["asym", "unsorted", "loop", "range", "dup"])
def test_bad_graph_rejected(Q, breakit, problem):
    g = gen.random_regular(50, 4, 1)
    rp, ci = g.rowptr.copy(), g.colidx.copy()
    if breakit == "asym":
        ci[0] = [j for j in range(50) if j not in ci[rp[0]:rp[1]] and j != 0][0]
        ci[rp[0]:rp[1]] = np.sort(ci[rp[0]:rp[1]])
    elif breakit == "unsorted":
        ci[rp[0]], ci[rp[0] + 1] = ci[rp[0] + 1], ci[rp[0]]
    elif breakit == "loop":
        ci[rp[3]] = 3
    elif breakit == "range":
        ci[rp[7]] = 10_000
    elif breakit == "dup":
        ci[rp[2] + 1] = ci[rp[2]]
    with pytest.raises(Q.QQAError) as e:   # every problem validates (the dense clique on the host)
        Q.Solver(rp, ci, Q.make_config(problem, S_total=8, **({"n_colors": 4} if problem == "coloring" else {})))
    assert e.value.status == 2


def test_bad_clique_batch_edge_rejected(Q):
    """Max clique on a batch: an edge joining two instances is rejected before the complement is built."""
    g0, g1 = gen.erdos_renyi(20, 0.5, 1), gen.erdos_renyi(20, 0.5, 2)
    g, gor = gen.disjoint_union([g0, g1])
    u, v = g.edges()
    u = np.append(u, 3)
    v = np.append(v, 25)
    bad = gen.from_edges(g.n, u, v)
    with pytest.raises(Q.QQAError) as e:
        Q.Solver(bad.rowptr, bad.colidx, Q.make_config("maxclique", S_total=8), group_of_row=gor)
    assert e.value.status == 2


def test_nonfinite_detected(Q):
    g = gen.random_regular(50, 4, 1)
    sol = gpu(Q, g, "mis", 8, 1, weight_decay=-1e38)
    sol.run_linear(-2.0, 0.1, 10)
    with pytest.raises(Q.QQAError) as e:
        sol.round_evaluate()
    assert e.value.status == 5


def test_degenerate_graphs(Q):
    # edgeless: every variable is free, MIS takes all of them
    g = gen.edgeless(37)
    sol = gpu(Q, g, "mis", 8, 1)
    sol.run_linear(-2.0, 0.1, 300)
    res = sol.round_evaluate()
    assert res.per_replica["size"].max() == 37 and res.best_energy == -37
    st = oracle.run(g, ocfg("mis", 8, 1), oracle.schedule(-2.0, 0.1, 300))
    assert_state_equal(sol, st)
    # single vertex, single edge
    for g in (gen.edgeless(1), gen.from_edges(2, [0], [1])):
        sol = gpu(Q, g, "maxcut", 4, 2)
        sol.run_linear(-5.0, 0.1, 100)
        st = oracle.run(g, ocfg("maxcut", 4, 2), oracle.schedule(-5.0, 0.1, 100))
        assert_state_equal(sol, st)
        assert sol.round_evaluate().best_energy == -g.n_edges


def test_empty_graph(Q):
    g = gen.edgeless(0)
    sol = gpu(Q, g, "mis", 4, 1)
    sol.run_linear(-2.0, 0.1, 5)
    res = sol.round_evaluate()
    assert res.best_energy == 0.0 and len(res.best_x) == 0


def test_nccl_single_rank_identical(Q):
    """The communicator path (one rank) gives exactly the no-communicator result."""
    g = gen.erdos_renyi(800, 0.02, 5)
    a = gpu(Q, g, "mis", 32, 8)
    b = gpu(Q, g, "mis", 32, 8)
    b.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 100, 0, 60)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k])
    ra, rb = a.round_evaluate(), b.round_evaluate()
    assert ra.best_replica == rb.best_replica and np.array_equal(ra.best_x, rb.best_x)


def test_profile_counts_launches(Q):
    g = gen.random_regular(1000, 8, 1)
    sol = gpu(Q, g, "mis", 64, 1)
    sol.profile(True)
    sol.run_linear(-2.0, 0.1, 100, 0, 25)
    ms, k = sol.profile_read()
    assert k == 25 and ms > 0


@pytest.mark.parametrize("SB", [8, 16, 32])
@pytest.mark.parametrize("problem,S", [("mis", 100), ("maxcut", 64), ("mis", 13), ("maxclique", 40)])
def test_replica_blocked_layout_parity(Q, monkeypatch, SB, problem, S):
    """Forced replica blocking ([B][n][SB], atomics across blocks) is bit-identical to the oracle."""
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", str(SB))
    g = gen.erdos_renyi(150, 0.5, 31) if problem == "maxclique" else gen.erdos_renyi(900, 0.02, 31)
    gam = oracle.schedule(-2.0, 0.1, 300)[:50]
    sol = gpu(Q, g, problem, S, 21, comm=0.3)
    sol.run(gam)
    st = oracle.run(g, ocfg(problem, S, 21, comm=0.3), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)
    counts, energy, best = oracle.evaluate(g, problem, 2.0, st.theta)
    res = sol.round_evaluate()
    assert np.array_equal(np.stack([res.per_replica["size"], res.per_replica["violations"],
                                    res.per_replica["cut"]], 1), counts)
    assert res.best_replica == best
    ck = sol.get_state()
    sol2 = gpu(Q, g, problem, S, 5, comm=0.3)
    sol2.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=sol.get_stats()["c"])
    assert np.array_equal(sol2.get_state()["p"], ck["p"])


@pytest.mark.parametrize("chunks", ["3", "7"])
def test_nccl_chunked_overlap_identical(Q, monkeypatch, chunks):
    """The compute / all-reduce overlap (rows in chunks, each chunk's sums all-reduced on a second
    stream while the next chunk computes) is bit-identical to the unchunked path."""
    monkeypatch.setenv("QQA_COMM_CHUNKS", chunks)
    g = gen.erdos_renyi(1000, 0.02, 5)
    a = gpu(Q, g, "maxcut", 24, 8, comm=0.5)
    b = gpu(Q, g, "maxcut", 24, 8, comm=0.5)
    b.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    b.profile(True)
    for s in (a, b):
        s.run_linear(-5.0, 0.1, 100, 0, 60)
    assert b.profile_read()[1] == 60                  # one timed span per step
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k])
    assert np.array_equal(a.get_stats()["sumD2"], b.get_stats()["sumD2"])


def test_share_comm(Q):
    """A second handle joins the first one's communicator; it survives the donor's destruction."""
    g = gen.erdos_renyi(600, 0.02, 6)
    a = gpu(Q, g, "mis", 16, 2)
    a.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    b = gpu(Q, g, "mis", 16, 2)
    b.share_comm(a)
    c = gpu(Q, g, "mis", 16, 2)
    a.close()
    for s in (b, c):
        s.run_linear(-2.0, 0.1, 100, 0, 40)
    for k in ("theta", "p"):
        assert np.array_equal(b.get_state()[k], c.get_state()[k])
    assert b.round_evaluate().best_replica == c.round_evaluate().best_replica


@pytest.mark.parametrize("problem,S,mp,T", [("mis", 16, "sigmoid", 0.0), ("maxcut", 100, "clamp", 0.001),
                                            ("maxclique", 40, "sigmoid", 0.001), ("mis", 256, "clamp", 0.0),
                                            ("mis", 3, "sigmoid", 0.0)])
def test_persistent_equals_launch_per_step(Q, monkeypatch, problem, S, mp, T):
    """The persistent cooperative kernel (one launch per <= 4096 steps, grid barrier per step)
    is bit-identical to one k_finalize + k_step launch per step, across a schedule-table chunk."""
    g = gen.erdos_renyi(150, 0.5, 12) if problem == "maxclique" else gen.erdos_renyi(700, 0.02, 12)
    steps = 4100 if S == 16 else 300
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("QQA_PERSISTENT", flag)
        sol = gpu(Q, g, problem, S, 4, map=mp, temperature=T)
        sol.profile(True)
        l0 = sol.launch_count()
        sol.run_linear(-2.0, 0.1, steps)
        launches = sol.launch_count() - l0
        assert sol.profile_read()[1] == steps
        out.append((sol.get_state(), sol.get_stats(), launches, sol.round_evaluate()))
    (a, sa, la, ra), (b, sb, lb, rb) = out
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("c", "sumD", "sumD2"):
        assert np.array_equal(sa[k], sb[k]), k
    assert ra.best_replica == rb.best_replica and np.array_equal(ra.best_x, rb.best_x)
    assert la == (steps + 4095) // 4096 and lb == 2 * steps


@pytest.mark.parametrize("cta", ["1024", "256"])
def test_persistent_cta_layouts_identical(Q, monkeypatch, cta):
    """Contiguous-row 1024-thread CTAs and strided 256-thread CTAs of the persistent kernel give the
    launch-per-step result bit for bit (c2-like batch of small instances)."""
    gs = [gen.erdos_renyi(300, 0.1, 60 + k) for k in range(6)]
    U, gor = gen.disjoint_union(gs)
    gam = oracle.schedule(-2.0, 0.1, 300)[:80]
    monkeypatch.setenv("QQA_RUN_CTA", cta)
    monkeypatch.setenv("QQA_PERSISTENT", "1")
    a = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=72, seed=3), group_of_row=gor)
    a.run(gam)
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    b = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=72, seed=3), group_of_row=gor)
    b.run(gam)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k


@pytest.mark.parametrize("name,path,SB", [("c1", "cluster", 16), ("c2", "persistent", 104), ("t1", "persistent", 104), ("c3", "persistent", 256), ("c4", "persistent", 512),
                                          ("c5", "step", 32), ("q13", "kary", 0)])
def test_step_path_and_replica_block(Q, name, path, SB):
    """Kernel selection of bench.py's workloads: c5's p (256 MB) exceeds the 128 MB
    block budget, so its 64 replicas run as two blocks of 32 (measured faster than unblocked)."""
    w = gen.workload(name)
    (g, gor) = w.batched()                      # bench.py's handle: the batch of a multi-instance workload
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config(w.problem, S_total=w.S, seed=w.seeds[0], **hp), group_of_row=gor)
    assert sol.step_path() == path and sol.replica_block() == SB


@pytest.mark.parametrize("problem,n,S,mp,T", [("mis", 256, 16, "sigmoid", 0.0), ("maxcut", 300, 100, "clamp", 0.001),
                                              ("maxclique", 60, 24, "sigmoid", 0.001), ("mis", 1000, 32, "clamp", 0.0),
                                              ("mis", 7, 3, "sigmoid", 0.0), ("maxcut", 2000, 13, "sigmoid", 0.001)])
def test_cluster_equals_launch_per_step(Q, monkeypatch, problem, n, S, mp, T):
    """The one-cluster shared-memory anneal (k_run_cluster: rows spread over the cluster's CTAs,
    neighbour rows through distributed shared memory, one cluster barrier per step) is bit-identical
    to one k_finalize + k_step launch per step, across a schedule-table chunk (4096 steps)."""
    g = gen.erdos_renyi(n, 0.5, 12) if problem == "maxclique" else gen.erdos_renyi(n, min(0.5, 6.0 / n), 12)
    steps = 4100 if (n, S) == (256, 16) else 300
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("QQA_CLUSTER", flag)
        monkeypatch.setenv("QQA_PERSISTENT", "0")
        sol = gpu(Q, g, problem, S, 4, map=mp, temperature=T, comm=0.3)
        assert sol.step_path() == ("cluster" if flag == "1" else "step")
        sol.profile(True)
        l0 = sol.launch_count()
        sol.run_linear(-2.0, 0.1, steps)
        launches = sol.launch_count() - l0
        assert sol.profile_read()[1] == steps
        out.append((sol.get_state(), sol.get_stats(), launches, sol.round_evaluate()))
    (a, sa, la, ra), (b, sb, lb, rb) = out
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("c", "sumD", "sumD2"):
        assert np.array_equal(sa[k], sb[k]), k
    assert ra.best_replica == rb.best_replica and np.array_equal(ra.best_x, rb.best_x)
    assert la == (steps + 4095) // 4096 and lb == 2 * steps


def test_cluster_then_resume_on_other_paths(Q, monkeypatch):
    """Buffers after a cluster run follow the k_run convention: continuing on k_step, or through a
    checkpoint, gives the uninterrupted result."""
    g = gen.random_regular(256, 3, 1)
    a = gpu(Q, g, "mis", 16, 9)
    assert a.step_path() == "cluster"
    a.run_linear(-2.0, 0.1, 400, 0, 150)
    monkeypatch.setenv("QQA_CLUSTER", "0")
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    a.run_linear(-2.0, 0.1, 400, 150, 151)     # one step: launch-per-step path
    monkeypatch.delenv("QQA_CLUSTER")
    monkeypatch.delenv("QQA_PERSISTENT")
    a.run_linear(-2.0, 0.1, 400, 151, 400)
    st = oracle.run(g, ocfg("mis", 16, 9), oracle.schedule(-2.0, 0.1, 400))
    assert_state_equal(a, st)
    assert_stats_equal(a, st)


STAGE_CASES = [
    # (problem, graph, S, hp, replica block)
    ("mis", lambda: gen.random_regular(3000, 20, 5), 64, dict(), "32"),                      # c5's layout
    ("mis", lambda: gen.random_regular(3000, 20, 5), 64, dict(), "16"),
    ("maxcut", lambda: gen.erdos_renyi(900, 0.02, 3), 64, dict(map="clamp", temperature=0.002, comm=0.5), None),
    ("mis", lambda: gen.erdos_renyi(700, 0.03, 4), 8, dict(alpha=4), None),
    ("maxcut", lambda: gen.random_regular(500, 5, 6), 256, dict(comm=1.0), None),
    ("mis", lambda: gen.erdos_renyi(800, 0.01, 7), 16, dict(map="clamp"), "8"),
]


@pytest.mark.parametrize("case", range(len(STAGE_CASES)))
def test_staged_state_kernel_parity(Q, monkeypatch, case):
    """k_step_st (round 2): the next item's theta / m / v / p staged in shared memory by cp.async while the
    current item updates -- the default for replica-blocked layouts; forced here on every FULL shape and the
    clamp / noise modes. Bit-exact against the contract oracle, like k_step."""
    problem, mk, S, hp, sb = STAGE_CASES[case]
    monkeypatch.setenv("QQA_STAGE", "1")
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    g = mk()
    gam = oracle.schedule(-2.0, 0.1, 500)[:50]
    sol = gpu(Q, g, problem, S, 13, **hp)
    assert sol.step_path() == "step"
    sol.run(gam)
    st = oracle.run(g, ocfg(problem, S, 13, **hp), gam)
    assert_state_equal(sol, st)
    assert_stats_equal(sol, st)


def test_serpentine_block_order_is_bit_identical(Q, monkeypatch):
    """QQA_SERPENTINE=1 sweeps the replica blocks in alternating order from step to step (an L2 experiment,
    DESIGN.md §4, off by default): the blocks meet only in exact int64 atomics, so the bits do not change."""
    g = gen.random_regular(2000, 20, 5)
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", "8")
    ref = gpu(Q, g, "mis", 40, 3)
    ref.run(oracle.schedule(-2.0, 0.1, 100)[:30])
    monkeypatch.setenv("QQA_SERPENTINE", "1")
    ser = gpu(Q, g, "mis", 40, 3)
    ser.run(oracle.schedule(-2.0, 0.1, 100)[:30])
    a, b = ref.get_state(), ser.get_state()
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
    assert np.array_equal(ref.get_stats()["sumD2"], ser.get_stats()["sumD2"])
