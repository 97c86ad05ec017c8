"""Fused statistics exchange (k_step_x, qqa_attach_exchange) on one GPU.

Each rank adds its replicas' fixed-point terms of row i into the OWNER rank's buffer inside the step
kernel and reads the owner's totals at the next step; step boundaries are an arrival-counter barrier
in the same buffers. On one device the G ranks are G shard handles on one stream, run in lockstep
(rank 0..G-1 for step t, then step t+1), so no kernel ever waits for a kernel queued behind it; the
peer "memory" is the other handles' buffers on the same GPU. The shards must reproduce the handle
holding every replica bit for bit, and the one-rank NCCL path. A rank that never arrives must be
reported, not hang. The concurrent tests run all G ranks at the same time in one cooperative launch
(qqa_exchange_emulate), so the barrier and the remote atomics are exercised under real concurrency.
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


def exchange_buffers(sols):
    import torch
    bufs = [torch.empty(s.exchange_bytes() + 256, dtype=torch.uint8, device=s.device) for s in sols]
    ptrs = [(b.data_ptr() + 255) // 256 * 256 for b in bufs]
    return bufs, ptrs


CASES = [("mis", 2, 32, dict(comm=0.3), None),
         ("maxcut", 4, 16, dict(comm=1.0, map="clamp", temperature=0.003), None),
         ("mis", 3, 13, dict(comm=0.5, temperature=0.002), None),          # odd offsets split noise pairs
         ("maxcut", 8, 8, dict(comm=0.1), None),                             # c5's shard size at 8 GPUs
         ("mis", 2, 40, dict(comm=0.3, alpha=4), "8"),                       # replica blocks: atomics per block
         ("maxclique", 2, 24, dict(comm=0.3), None)]                        # dense complement


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fused_exchange_shards_reproduce_the_full_ensemble(Q, monkeypatch, case):
    problem, G, S_l, hp, sb = CASES[case]
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    g = gen.erdos_renyi(120, 0.5, 7) if problem == "maxclique" else gen.erdos_renyi(501, 0.03, 40 + case)
    S = G * S_l
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 400)[:60]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, **hp))
    full.run(gam)
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs)
        assert sh.step_path() == "exchange"
    Q.loopback_sync_init(shards)            # initial totals into every shard, then the first barrier
    Q.loopback_run(shards, gam[:25])        # lockstep, no host-side reduction: exchanged in-kernel
    for t in range(25, 60):                 # single steps through the public run() as well
        for sh in shards:
            sh.run(gam[t:t + 1])
    fs, fst = full.get_state(), full.get_stats()
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
        st = sh.get_stats()                  # owner rows gathered from every rank's buffer
        for f in ("c", "sumD", "sumD2"):
            assert np.array_equal(st[f], fst[f]), (r, f)
    fr = full.round_evaluate().per_replica
    for r, sh in enumerate(shards):
        pr = sh.round_evaluate().per_replica
        for f in ("size", "violations", "cut", "energy"):
            assert np.array_equal(pr[f], fr[f][r * S_l:(r + 1) * S_l]), (r, f)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fused_exchange_concurrent_ranks_reproduce_the_full_ensemble(Q, monkeypatch, case):
    """The same shards, but the G ranks run CONCURRENTLY: one cooperative launch (qqa_exchange_emulate) whose
    grid is G slices of co-resident CTAs, so every rank's step really waits on the other ranks' arrivals
    (red.release.sys / ld.acquire.sys barrier) and their remote atomics race with its own -- the multi-GPU
    protocol under real concurrency on one device. Bit-exact against the handle holding all replicas."""
    problem, G, S_l, hp, sb = CASES[case]
    if sb:
        monkeypatch.setenv("QQA_BLOCK_REPLICAS", sb)
    g = gen.erdos_renyi(120, 0.5, 7) if problem == "maxclique" else gen.erdos_renyi(501, 0.03, 40 + case)
    S = G * S_l
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 400)[:60]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, **hp))
    full.run(gam)
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs)
    Q.loopback_sync_init(shards)
    Q.exchange_emulate(shards, gam[:35])     # concurrent ranks, 35 steps in one launch
    for t in range(35, 60):                  # then the production per-step launches continue from there
        for sh in shards:
            sh.run(gam[t:t + 1])
    fs, fst = full.get_state(), full.get_stats()
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        assert ss["step"] == 60
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
        st = sh.get_stats()
        for f in ("c", "sumD", "sumD2"):
            assert np.array_equal(st[f], fst[f]), (r, f)
    fr = full.round_evaluate().per_replica
    for r, sh in enumerate(shards):
        pr = sh.round_evaluate().per_replica
        for f in ("size", "violations", "cut", "energy"):
            assert np.array_equal(pr[f], fr[f][r * S_l:(r + 1) * S_l]), (r, f)


def test_fused_exchange_concurrent_c5_shards(Q):
    """c5's graph (20-regular, N = 1e6) split as 8 concurrent ranks of 8 replicas (the G = 8 shard of the
    scaling run): 20 steps in one cooperative launch, bit-exact against one handle with all 64 replicas."""
    w = gen.workload("c5")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:20]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=64, seed=w.seeds[0], **hp))
    full.run(gam)
    fs = full.get_state()
    fst = full.get_stats()
    full.close()
    G, S_l = 8, 8
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=64, seed=w.seeds[0], replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs)
    Q.loopback_sync_init(shards)
    Q.exchange_emulate(shards, gam)
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        for f in ("theta", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
    st = shards[3].get_stats()
    assert np.array_equal(st["sumD2"], fst["sumD2"]) and np.array_equal(st["c"], fst["c"])


def test_fused_exchange_one_rank_equals_nccl(Q):
    """One rank with a real (one-rank) NCCL communicator: the fused path (own buffer as the only peer)
    equals the NCCL all-reduce path, across reset and checkpoint resume."""
    import torch
    g = gen.random_regular(3000, 20, 5)
    mk = lambda: Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=64, seed=3, comm=0.2))
    a, b = mk(), mk()
    for s in (a, b):
        s.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    buf = torch.empty(b.exchange_bytes(), dtype=torch.uint8, device=b.device)
    b.attach_exchange([buf.data_ptr()], 0, 1, keep=buf)
    assert a.step_path() == "step" and b.step_path() == "exchange"
    for s in (a, b):
        s.reset()
        s.run_linear(-2.0, 0.1, 300, 0, 80)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k
    for k in ("c", "sumD", "sumD2"):
        assert np.array_equal(a.get_stats()[k], b.get_stats()[k]), k
    ra, rb = a.round_evaluate(), b.round_evaluate()
    assert ra.best_replica == rb.best_replica and np.array_equal(ra.best_x, rb.best_x)
    ck, cs = b.get_state(), b.get_stats()
    b.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=cs["c"])
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 300, 80, 120)
    for k in ("theta", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k


def test_fused_exchange_missing_peer_is_reported_not_hung(Q):
    """Rank 1 never runs its step: rank 0's step kernel gives up waiting at the barrier after a
    bounded spin and the next synchronising call reports QQA_ERR_COMM."""
    g = gen.erdos_renyi(200, 0.05, 3)
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=16, seed=1, replica_offset=8 * r,
                                                         S_local=8)) for r in range(2)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, 2, keep=bufs)
    Q.loopback_sync_init(shards)
    gam = oracle.schedule(-2.0, 0.1, 10)
    shards[0].run(gam[:1])                  # barrier of step 0 complete: fine
    shards[0].run(gam[1:2])                 # rank 1 never arrived for step 0 -> bounded wait, flagged
    with pytest.raises(Q.QQAError, match="never arrived"):
        shards[0].round_evaluate()


def test_fused_exchange_rejects_unsupported(Q):
    g = gen.queens(5, 5)
    k = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=8, seed=1, n_colors=5))
    with pytest.raises(Q.QQAError):
        k.attach_exchange([1 << 20], 0, 1)
    g2 = gen.erdos_renyi(100, 0.05, 1)
    s = Q.Solver(g2.rowptr, g2.colidx, Q.make_config("mis", S_total=16, seed=1, replica_offset=0, S_local=8))
    with pytest.raises(Q.QQAError):
        s.attach_exchange([1 << 20], 1, 2)    # replica_offset 0 is rank 0's shard


@pytest.mark.parametrize("mode", ["auto", "fused", "slotted"])
def test_bench_multi_gpu_code_path_at_one_rank(Q, mode):
    """bench.py's N > 1 code path (process group, NCCL communicator, symmetric-memory exchange buffers,
    self-check and speed probe) at one rank: exactly one JSON line on stdout, the exchange recorded."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "c3", "--force-dist",
                          "--exchange", mode, "--no-cpu", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0
    if mode in ("fused", "slotted"):
        assert d["config"]["exchange"].startswith("fused") and d["roofline"]["kernel"].startswith("qqa::k_step_x")
        assert ("slotted" in d["config"]["exchange"]) == (mode == "slotted")
    else:   # c3 has one replica block: both fused modes pass the self-check and are timed beside NCCL
        probe = d["config"]["exchange_probe"]
        assert probe["nccl_ms_per_step"] > 0 and probe["atomic_ms_per_step"] > 0 and probe["slotted_ms_per_step"] > 0


@pytest.mark.parametrize("kind,problem,G,S_l,hp", [("pm1", "maxcut", 4, 16, dict(comm=0.3)),
                                                   ("int", "mis", 2, 32, dict(comm=0.5, map="clamp", temperature=0.002)),
                                                   ("uniform", "maxcut", 8, 8, dict(comm=0.1))])
def test_fused_exchange_weighted_graphs(Q, kind, problem, G, S_l, hp):
    """Edge-weighted graphs (Optsicom +-1 weights) through the fused exchange, ranks run in lockstep
    and then concurrently (one cooperative launch): bit-identical to the handle holding every replica."""
    g = gen.with_weights(gen.erdos_renyi(400, 0.03, 11), kind, 5)
    S = G * S_l
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 300)[:40]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=3, **hp), weights=g.weights)
    full.run(gam)
    fs, fst = full.get_state(), full.get_stats()
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=3, replica_offset=r * S_l,
                                                         S_local=S_l, **hp), weights=g.weights) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs)
    Q.loopback_sync_init(shards)
    Q.loopback_run(shards, gam[:20])        # lockstep
    Q.exchange_emulate(shards, gam[20:])    # concurrent
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
        st = sh.get_stats()
        for f in ("c", "sumD", "sumD2"):
            assert np.array_equal(st[f], fst[f]), (r, f)
    fr = full.round_evaluate().per_replica
    for r, sh in enumerate(shards):
        pr = sh.round_evaluate().per_replica
        for f in ("wviolations", "wcut", "energy"):
            assert np.array_equal(pr[f], fr[f][r * S_l:(r + 1) * S_l]), (r, f)


def test_detach_exchange_returns_to_the_nccl_path(Q):
    """qqa_detach_exchange (bench.py's fallback when a rank cannot run the fused exchange): after a fused run,
    detach + reset gives a handle on the NCCL path that reproduces a plain NCCL handle bit for bit."""
    import torch
    g = gen.random_regular(2000, 10, 2)
    mk = lambda: Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=32, seed=4, comm=0.2))
    a, b = mk(), mk()
    for s in (a, b):
        s.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    buf = torch.empty(b.exchange_bytes(), dtype=torch.uint8, device=b.device)
    b.attach_exchange([buf.data_ptr()], 0, 1, keep=buf)
    b.run_linear(-2.0, 0.1, 100, 0, 10)
    b.detach_exchange()
    assert b.step_path() != "exchange"
    b.reset()
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 100, 0, 40)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k
    for k in ("c", "sumD", "sumD2"):
        assert np.array_equal(a.get_stats()[k], b.get_stats()[k]), k


SLOT_CASES = [c for c in CASES if c[4] is None]   # the owner-slotted exchange needs one replica block


@pytest.mark.parametrize("case", range(len(SLOT_CASES)))
def test_slotted_exchange_concurrent_ranks_reproduce_the_full_ensemble(Q, case):
    """Owner-slotted exchange (qqa_attach_exchange_mode SLOTTED): partials stored into per-writer slots at the
    owner, owner-side sum after a barrier, totals read after a second barrier -- no remote atomics. G ranks
    run concurrently in one cooperative launch (the mid-kernel barrier needs every rank resident); bit-exact
    against the handle holding every replica, including the statistics and the evaluation."""
    problem, G, S_l, hp, _ = SLOT_CASES[case]
    g = gen.erdos_renyi(120, 0.5, 7) if problem == "maxclique" else gen.erdos_renyi(501, 0.03, 40 + case)
    S = G * S_l
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 400)[:60]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, **hp))
    full.run(gam)
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs, mode="slotted")
    Q.loopback_sync_init(shards)            # every buffer zeroed: scatter the initial partials, first barrier
    st0 = shards[1].get_stats()             # the initial totals, gathered from the owners' slots
    f0 = Q.Solver(g.rowptr, g.colidx, Q.make_config(problem, S_total=S, seed=9, **hp)).get_stats()
    assert np.array_equal(st0["sumD"], f0["sumD"]) and np.array_equal(st0["sumD2"], f0["sumD2"])
    Q.exchange_emulate(shards, gam[:25])
    Q.exchange_emulate(shards, gam[25:])
    fs, fst = full.get_state(), full.get_stats()
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        assert ss["step"] == 60
        for f in ("theta", "m", "v", "p"):
            assert np.array_equal(ss[f].view(np.uint32), fs[f][:, r * S_l:(r + 1) * S_l].view(np.uint32)), (r, f)
        st = sh.get_stats()
        for f in ("c", "sumD", "sumD2"):
            assert np.array_equal(st[f], fst[f]), (r, f)
    fr = full.round_evaluate().per_replica
    for r, sh in enumerate(shards):
        pr = sh.round_evaluate().per_replica
        for f in ("size", "violations", "cut", "energy"):
            assert np.array_equal(pr[f], fr[f][r * S_l:(r + 1) * S_l]), (r, f)


def test_slotted_exchange_c5_shards_and_one_rank_nccl(Q):
    """c5's graph as 8 concurrent slotted ranks (20 steps), and one rank with a real NCCL communicator on the
    production launch (cooperative k_step_xs per step) across reset and resume: both bit-exact."""
    import torch
    w = gen.workload("c5")
    g = w.graphs[0]
    hp = {k: v for k, v in w.hparams().items() if k != "problem"}
    gam = oracle.schedule(w.gamma_min, w.gamma_max, w.steps)[:20]
    full = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=64, seed=w.seeds[0], **hp))
    full.run(gam)
    fs = full.get_state()
    full.close()
    G, S_l = 8, 8
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=64, seed=w.seeds[0], replica_offset=r * S_l,
                                                         S_local=S_l, **hp)) for r in range(G)]
    bufs, ptrs = exchange_buffers(shards)
    for r, sh in enumerate(shards):
        sh.attach_exchange(ptrs, r, G, keep=bufs, mode="slotted")
    Q.loopback_sync_init(shards)            # every buffer zeroed: scatter the initial partials, first barrier
    Q.exchange_emulate(shards, gam)
    for r, sh in enumerate(shards):
        ss = sh.get_state()
        assert np.array_equal(ss["theta"].view(np.uint32), fs["theta"][:, r * S_l:(r + 1) * S_l].view(np.uint32)), r
    for sh in shards:
        sh.close()
    del shards, bufs
    g2 = gen.random_regular(3000, 20, 5)
    mk = lambda: Q.Solver(g2.rowptr, g2.colidx, Q.make_config("mis", S_total=32, seed=3, comm=0.2))
    a, b = mk(), mk()
    for s in (a, b):
        s.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    buf = torch.empty(b.exchange_bytes(), dtype=torch.uint8, device=b.device)
    b.attach_exchange([buf.data_ptr()], 0, 1, keep=buf, mode="slotted")
    assert b.step_path() == "exchange"
    for s in (a, b):
        s.reset()
        s.run_linear(-2.0, 0.1, 300, 0, 60)
    for k in ("theta", "m", "v", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k
    for k in ("c", "sumD", "sumD2"):
        assert np.array_equal(a.get_stats()[k], b.get_stats()[k]), k
    ra, rb = a.round_evaluate(), b.round_evaluate()
    assert ra.best_replica == rb.best_replica and np.array_equal(ra.best_x, rb.best_x)
    ck, cs = b.get_state(), b.get_stats()
    b.set_state(ck["theta"], ck["m"], ck["v"], ck["step"], c=cs["c"])
    for s in (a, b):
        s.run_linear(-2.0, 0.1, 300, 60, 90)
    for k in ("theta", "p"):
        assert np.array_equal(a.get_state()[k], b.get_state()[k]), k


def test_slotted_exchange_rejects_replica_blocks(Q, monkeypatch):
    monkeypatch.setenv("QQA_BLOCK_REPLICAS", "8")
    g = gen.erdos_renyi(200, 0.05, 1)
    s = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=32, seed=1, replica_offset=0, S_local=16))
    with pytest.raises(Q.QQAError) as e:
        s.attach_exchange([1 << 20, 2 << 20], 0, 2, mode="slotted")
    assert e.value.status == 6
