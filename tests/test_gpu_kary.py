"""GPU parity for NEXT-4 (K-ary PQQA / graph colouring, App. B, map P:672-676,
energy P:745-750) through the C ABI, against the fp32 contract oracle: P, m, v and the
per-(variable, colour) statistics bit-identical; colours, conflicts, energies and the
best replica bit-exact."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_02135_b200 as Q
    return Q


def gpu(Q, g, K, S, seed, S_total=None, offset=0, **hp):
    cfg = Q.make_config("coloring", S_total=S if S_total is None else S_total, seed=seed, replica_offset=offset,
                        S_local=S, n_colors=K, **hp)
    return Q.Solver(g.rowptr, g.colidx, cfg)


def ocfg(S, seed, **hp):
    return oracle.make_cfg("mis", S=S, seed=seed, threads=8, **hp)


def assert_equal_K(sol, st):
    gs = sol.get_state()
    for f, ref in (("p", st.P), ("theta", st.P), ("m", st.m), ("v", st.v)):
        bad = np.count_nonzero(gs[f].view(np.uint32) != ref.view(np.uint32))
        assert bad == 0, f"{f}: {bad} of {ref.size} differ (max |d| = {np.abs(gs[f] - ref).max()})"
    ss = sol.get_stats()
    assert np.array_equal(ss["c"].view(np.uint32), st.c.view(np.uint32))
    assert np.array_equal(ss["sumD"], st.sumD) and np.array_equal(ss["sumD2"], st.sumD2)


@pytest.mark.parametrize("K", [2, 3, 5, 9, 13, 16])
@pytest.mark.parametrize("S", [1, 7, 32, 100])
def test_init_parity(Q, K, S):
    g = gen.queens(5, 5)
    sol = gpu(Q, g, K, S, 17)
    assert_equal_K(sol, oracle.init_K(g, ocfg(S, 17), K))


CASES = [
    # (graph, K, S, hyper-parameters)
    (lambda: gen.queens(5, 5), 5, 16, dict(lr=0.1)),
    (lambda: gen.mycielski(5), 6, 100, dict(lr=0.1)),
    (lambda: gen.erdos_renyi(300, 0.03, 6), 3, 64, dict(lr=0.1, temperature=0.001, comm=0.3)),
    (lambda: gen.queens(8, 8), 9, 33, dict(lr=0.1, comm=0.3, alpha=4)),
    (lambda: gen.random_regular(500, 8, 2), 16, 8, dict(lr=0.03)),
    (lambda: gen.grid(10, 12), 2, 40, dict(lr=0.1, temperature=0.01)),
    (lambda: gen.erdos_renyi(200, 0.05, 9), 4, 1, dict(lr=0.1)),
]


@pytest.mark.parametrize("kary_grad", [1, 0])   # gradient through the map (R33, default) / dR/dP (R29)
@pytest.mark.parametrize("case", range(len(CASES)))
def test_fifty_steps_parity(Q, case, kary_grad):
    mk, K, S, hp = CASES[case]
    hp = dict(hp, kary_grad=kary_grad)
    g = mk()
    gam = oracle.schedule(-2.0, 0.1, 1000)[:50]
    sol = gpu(Q, g, K, S, 11, **hp)
    sol.run(gam)
    st = oracle.run_K(g, ocfg(S, 11, **hp), K, gam)
    assert_equal_K(sol, st)


@pytest.mark.parametrize("name,K", [("queen5-5", 5), ("myciel5", 6)])
def test_full_schedule_with_evaluation(Q, name, K):
    """3000 steps at S=100 (the oracle finds a proper colouring for both, Table 4 reports 0 conflicts):
    state, colours, conflicts and the best replica bit-exact; best replica conflict-free."""
    g = gen.queens(5, 5) if name == "queen5-5" else gen.mycielski(5)
    sol = gpu(Q, g, K, 100, 1, lr=0.1)
    sol.run_linear(-2.0, 0.1, 3000)
    st = oracle.run_K(g, ocfg(100, 1, lr=0.1), K, oracle.schedule(-2.0, 0.1, 3000))
    assert_equal_K(sol, st)
    counts, energy, best, X = oracle.evaluate_K(g, st.P)
    res = sol.round_evaluate()
    pr = res.per_replica
    assert np.array_equal(pr["violations"], counts[:, 1]) and np.array_equal(pr["cut"], counts[:, 2])
    assert np.array_equal(pr["energy"], energy) and res.best_replica == best
    assert np.array_equal(res.best_x, X[:, best]) and res.best_energy == 0
    assert pr["feasible"][best] == 1


def test_checkpoint_resume(Q):
    g = gen.queens(6, 6)
    gam = oracle.schedule(-2.0, 0.1, 200)
    a = gpu(Q, g, 7, 24, 5, lr=0.1, temperature=0.001)
    a.run(gam[:30])
    ck, cs = a.get_state(), a.get_stats()
    a.run(gam[30:60])
    b = gpu(Q, g, 7, 24, 5, lr=0.1, temperature=0.001)   # same seed: the noise stream is keyed by it
    b.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=cs["c"])
    assert np.array_equal(b.get_stats()["sumD"], cs["sumD"])
    b.run(gam[30:60])
    for f in ("p", "m", "v"):
        assert np.array_equal(a.get_state()[f], b.get_state()[f])


def test_shard_is_column_slice_without_comm(Q):
    g = gen.queens(5, 5)
    gam = oracle.schedule(-2.0, 0.1, 100)[:40]
    full = gpu(Q, g, 5, 64, 3, comm=0.0, lr=0.1, temperature=0.01)
    full.run(gam)
    fs = full.get_state()
    for off, S in [(0, 32), (32, 32), (8, 8)]:
        sh = gpu(Q, g, 5, S, 3, S_total=64, offset=off, comm=0.0, lr=0.1, temperature=0.01)
        sh.run(gam)
        assert np.array_equal(sh.get_state()["p"], fs["p"][:, off:off + S])


def test_invalid_colouring_configs(Q):
    g = gen.queens(4, 4)
    for K in (0, 1, 17):
        with pytest.raises(Q.QQAError) as e:
            gpu(Q, g, K, 8, 1)
        assert e.value.status == 1
    U, gor = gen.disjoint_union([g, g])
    with pytest.raises(Q.QQAError) as e:
        Q.Solver(U.rowptr, U.colidx, Q.make_config("coloring", S_total=8, n_colors=4), group_of_row=gor)
    assert e.value.status == 6
    for kg in (-1, 2):
        with pytest.raises(Q.QQAError) as e:
            gpu(Q, g, 4, 8, 1, kary_grad=kg)
        assert e.value.status == 1


@pytest.mark.parametrize("kary_grad", [1, 0])
@pytest.mark.parametrize("K,S,T,steps", [(13, 1000, 0.0, 40), (10, 37, 0.002, 60), (16, 8, 0.0, 30), (9, 100, 0.001, 4100),
                                         (8, 64, 0.0, 40), (6, 37, 0.002, 60), (7, 100, 0.001, 4100), (8, 5, 0.0, 30)])
def test_colour_quad_kernel_equals_k_step_K(Q, monkeypatch, K, S, T, steps, kary_grad):
    """k_step_Kq (4 colours per thread; KP = 12 / 16: 4 lanes per replica, 8 replicas per warp; KP = 8 with
    QQA_KARY_QUAD=2: 2 lanes per replica, 16 replicas per warp) is bit-identical to k_step_K,
    including noise pairs, ragged replica chunks and a schedule longer than one run() call."""
    g = gen.queens(7, 7)
    out = []
    for flag in ("2", "0"):
        monkeypatch.setenv("QQA_KARY_QUAD", flag)
        sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=S, seed=3, n_colors=K, lr=0.01,
                                                         temperature=T, comm=0.3, kary_grad=kary_grad))
        sol.run_linear(-2.0, 0.1, steps)
        out.append((sol.get_state(), sol.get_stats(), sol.round_evaluate()))
    (a, sa, ra), (b, sb, rb) = out
    for f in ("theta", "m", "v", "p"):
        assert np.array_equal(a[f].view(np.uint32), b[f].view(np.uint32)), f
    for f in ("c", "sumD", "sumD2"):
        assert np.array_equal(sa[f], sb[f]), f
    assert ra.best_replica == rb.best_replica


def test_gradient_through_the_map_reaches_table_4_on_small_queens(Q):
    """Reading R33 on the GPU path: queen6-6 (7 colours), queen7-7 (7), queen8-8 (9) and queen9-9 (10)
    coloured without a conflict, as Table 4 reports for PQQA."""
    for (r, K) in [(6, 7), (7, 7), (8, 9), (9, 10)]:
        g = gen.queens(r, r)
        sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=1000, seed=1, n_colors=K, lr=0.1,
                                                         temperature=0.001))
        sol.run_linear(-2.0, 0.1, 3000)
        assert int(sol.round_evaluate().best_energy) == 0, (r, K)


@pytest.mark.parametrize("K,S", [(8, 64), (13, 100), (5, 9)])
def test_item_order_and_chunk_width_do_not_change_results(Q, monkeypatch, K, S):
    """Round 2 walks (replica chunk, variable) items chunk-major with chunks narrowed to fit L2;
    the per-(variable, colour) statistics meet in exact int64 atomics, so every order and chunk width gives the
    same bits, and the contract oracle's."""
    g = gen.random_regular(600, 8, 4)
    gam = oracle.schedule(-2.0, 0.1, 200)[:40]
    hp = dict(lr=0.01, comm=0.3)
    st = oracle.run_K(g, ocfg(S, 21, **hp), K, gam)
    for cmaj in ("0", "1"):
        for lanes in ("4", "8", "32"):
            monkeypatch.setenv("QQA_KARY_CMAJ", cmaj)
            monkeypatch.setenv("QQA_KARY_LANES", lanes)
            monkeypatch.setenv("QQA_KARY_QUAD", "0")   # k_step_K itself for every K (the quad kernel: KP 12 / 16)
            sol = gpu(Q, g, K, S, 21, **hp)
            sol.run(gam)
            assert_equal_K(sol, st)
            sol.close()


@pytest.mark.parametrize("name,steps", [("k8", 30), ("q13", 30)])
def test_bench_colouring_workloads_full_size(Q, name, steps):
    """The K-ary bench workloads at full size in bench.py's launch configuration (k8: N = 1e5, K = 8, S = 64,
    chunk-major items narrowed to 8-replica chunks; q13: queen13-13, K = 13, S = 1000, colour-quad kernel):
    P, m, v and the per-(variable, colour) statistics bit-exact after `steps` steps, then colours and
    conflicts of every replica bit-exact."""
    w = gen.workload(name)
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k not in ("problem", "n_colors")}
    cfg = Q.make_config("coloring", S_total=w.S, seed=w.seeds[0], n_colors=w.n_colors, **hp)
    sol = Q.Solver(g.rowptr, g.colidx, cfg)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, steps)
    ohp = {k: v for k, v in hp.items() if k not in ("map",)}
    st = oracle.run_K(g, oracle.make_cfg("mis", S=w.S, seed=w.seeds[0], threads=16, **ohp), w.n_colors,
                      oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:steps])
    assert_equal_K(sol, st)
    counts, energy, best, X = oracle.evaluate_K(g, st.P)
    res = sol.round_evaluate()
    assert np.array_equal(res.per_replica["violations"], counts[:, 1])
    assert res.best_replica == best
