"""T5 of SURVEY.md §4: the sharded multi-GPU semantics on ONE GPU. G replica shards of one ensemble are
G handles on one device and stream; the loopback exchange adds their int64 statistic sums after every
step exactly as the per-step NCCL all-reduce does across GPUs (no kernel waits on another). The shards
must reproduce one handle holding all replicas bit for bit -- replica offsets, the global-replica-keyed
init and noise (including pairs split by odd offsets), blocked layouts and the K-ary statistics."""
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


CASES = [("mis", 2, 32, dict(comm=0.3), None),
         ("maxcut", 4, 16, dict(comm=1.0, map="clamp", temperature=0.003), None),
         ("mis", 3, 13, dict(comm=0.5, temperature=0.002), None),          # odd offsets split noise pairs
         ("maxcut", 8, 8, dict(comm=0.1), None),                             # c5's shard size at 8 GPUs
         ("mis", 2, 40, dict(comm=0.3, alpha=4), "8"),                       # replica-blocked layout
         ("coloring", 4, 10, dict(comm=0.2, n_colors=5, lr=0.1, temperature=0.002), None),
         ("maxclique_sparse", 2, 24, dict(comm=0.3), None)]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_shards_reproduce_the_full_ensemble(Q, monkeypatch, case):
    problem, G, S_l, hp, sb = CASES[case]
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    g = gen.queens(6, 6) if problem == "coloring" else gen.erdos_renyi(500, 0.03 if problem != "maxclique_sparse" else 0.3, 40 + case)
    S = G * S_l
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 400)[:60]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, **hp))
    full.run(gam)
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    Q.loopback_sync_init(shards)
    Q.loopback_run(shards, gam)
    fs, fst = full.get_state(), full.get_stats()
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
        st = sh.get_stats()
        for f in ("c", "sumD", "sumD2"):
            assert np.array_equal(st[f], fst[f]), (r, f)
    # per-replica evaluation of each shard equals the full run's columns
    fr = full.round_evaluate().per_replica
    for r, sh in enumerate(shards):
        pr = sh.round_evaluate().per_replica
        for f in ("size", "violations", "cut", "energy"):
            assert np.array_equal(pr[f], fr[f][r * S_l:(r + 1) * S_l]), (r, f)


def test_loopback_rejects_inconsistent_shards(Q):
    g = gen.erdos_renyi(100, 0.05, 1)
    a = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=16, seed=1, replica_offset=0, S_local=8))
    b = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=16, seed=1, replica_offset=0, S_local=8))
    with pytest.raises(Q.QQAError):
        Q.loopback_sync_init([a, b])        # shard 1 must start at offset 8
