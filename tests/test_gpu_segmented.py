"""GPU parity of the segmented gather (round 2; QQA_SEGMENTS=KS).

The sources j of a replica block are split into KS ascending ranges; launch (b, k) adds the neighbours in
segment k to a partial q_i kept in the item's p_next row, the last launch adds the last segment and does the
update. Each row's neighbours are strictly ascending (k_validate), so the adds happen in CSR order and the
result must be bit-identical to the one-pass k_step -- and so to the fp32 contract oracle.
"""
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


def _solver(Q, g, problem, S, seed, **hp):
    cfg = Q.make_config(problem, S_total=S, seed=seed, S_local=S, **hp)
    return Q.Solver(g.rowptr, g.colidx, cfg)


def _assert_bits(sol, st):
    gs = sol.get_state()
    for k in ("theta", "m", "v", "p"):
        bad = np.count_nonzero(gs[k].view(np.uint32) != getattr(st, k).view(np.uint32))
        assert bad == 0, f"{k}: {bad} of {gs[k].size} elements differ bitwise"
    s = sol.get_stats()
    assert np.array_equal(s["c"].view(np.uint32), st.c.view(np.uint32))
    assert np.array_equal(s["sumD"], st.sumD)
    assert np.array_equal(s["sumD2"], st.sumD2)


CASES = [
    # problem, graph, S, hyper-parameters, QQA_BLOCK_REPLICAS, QQA_SEGMENTS
    ("mis", lambda: gen.random_regular(2000, 20, 5), 64, dict(), "32", "2"),       # c5's shape: 2 blocks of 32
    ("mis", lambda: gen.random_regular(2000, 20, 5), 64, dict(), "32", "3"),
    ("mis", lambda: gen.random_regular(2000, 20, 5), 64, dict(comm=0.3), "16", "5"),
    ("maxcut", lambda: gen.erdos_renyi(900, 0.02, 3), 64, dict(map="clamp", temperature=0.002, comm=0.5), "16", "3"),
    ("mis", lambda: gen.erdos_renyi(700, 0.03, 4), 8, dict(alpha=4, temperature=0.001), None, "4"),
    ("maxcut", lambda: gen.random_regular(500, 5, 6), 256, dict(comm=1.0), None, "2"),
    ("mis", lambda: gen.erdos_renyi(800, 0.002, 7), 16, dict(map="clamp"), "8", "7"),   # many empty (row, segment)
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_segmented_gather_bit_exact(Q, monkeypatch, case):
    problem, mk, S, hp, sb, ks = CASES[case]
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    monkeypatch.setenv("QQA_SEGMENTS", ks)
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    g = mk()
    gam = oracle.schedule(-2.0, 0.1, 500)[:50]
    sol = _solver(Q, g, problem, S, 13, **hp)
    assert sol.step_path() == "step"
    B = (S + 7) // 8 * 8 // int(sb) if sb else 1
    l0 = sol.launch_count()
    sol.run(gam[:1])
    assert sol.launch_count() - l0 == 1 + B * int(ks)    # finalize + KS passes per block: the segmented path ran
    sol.run(gam[1:])
    st = oracle.run(g, oracle.make_cfg(problem, S=S, seed=13, threads=8, **hp), gam)
    _assert_bits(sol, st)
    counts, energy, best = oracle.evaluate(g, problem, 2.0, st.theta, map=hp.get("map", "sigmoid"))
    res = sol.round_evaluate()
    assert np.array_equal(np.stack([res.per_replica["size"], res.per_replica["violations"],
                                    res.per_replica["cut"]], 1), counts)
    assert res.best_replica == best


@pytest.mark.parametrize("chunks", ["1", "3"])
def test_segmented_with_nccl_chunks_identical(Q, monkeypatch, chunks):
    """One-rank communicator: the all-reduce path (its last pass split into row chunks overlapped with the
    all-reduce) with segments equals the unsegmented handle bit for bit."""
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", "16")
    monkeypatch.setenv("QQA_COMM_CHUNKS", chunks)
    g = gen.random_regular(3000, 20, 9)
    a = _solver(Q, g, "mis", 48, 4, comm=0.2)
    monkeypatch.setenv("QQA_SEGMENTS", "3")
    b = _solver(Q, g, "mis", 48, 4, comm=0.2)
    b.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 200, 0, 40)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k].view(np.uint32), b.get_state()[k].view(np.uint32)), k
    assert np.array_equal(a.get_stats()["sumD2"], b.get_stats()["sumD2"])


def test_segments_ignored_where_unsupported(Q, monkeypatch):
    """Weighted graphs, VPL > 1 shapes and tiny graphs keep the one-pass kernel (same bits, 1 launch per step)."""
    monkeypatch.setenv("QQA_PERSISTENT", "0")
    monkeypatch.setenv("QQA_SEGMENTS", "4")
    g = gen.random_regular(400, 6, 2)
    sol = _solver(Q, g, "mis", 512, 3)      # S_p = 512: VPL = 2
    l0 = sol.launch_count()
    sol.run(oracle.schedule(-2.0, 0.1, 10)[:2])
    assert sol.launch_count() - l0 == 2 * 2

