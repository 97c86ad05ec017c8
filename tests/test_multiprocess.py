"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The GPU exchange is one all-reduce of the 2n int64 replica-statistic sums per
step. These tests run the same decomposition on the CPU: each
rank computes the fixed-point sums of its replica shard (the contract of
DESIGN.md §3), the ranks all-reduce them over gloo, and the result must equal
the unsharded sums exactly -- which is what makes any GPU count bit-identical.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fixed_point_sums(P, c):
    d = (P - c[:, None]).astype(np.float32)
    D = np.rint((d * np.float32(2.0 ** 40)).astype(np.float64)).astype(np.int64).sum(axis=1)
    dd = (d * d).astype(np.float32)
    D2 = np.rint((dd * np.float32(2.0 ** 40)).astype(np.float64)).astype(np.int64).sum(axis=1)
    return D, D2


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_02135_b200 import dist as qdist
    try:
        S = 24
        off, S_l = qdist.shard(S, world, rank)
        # the full ensemble (what every rank would hold at G = 1)
        g = gen.random_regular(200, 4, 3)
        st = oracle.run(g, oracle.make_cfg("mis", S=S, seed=9), oracle.schedule(-2.0, 0.1, 100)[:7])
        c = st.c
        # this rank's shard -> partial sums -> all-reduce
        D, D2 = _fixed_point_sums(st.p[:, off:off + S_l], c)
        t = torch.from_numpy(np.stack([D, D2]))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        full = t.numpy()
        np.save(os.path.join(out_dir, f"sums_{rank}.npy"), full)
        np.save(os.path.join(out_dir, "ref.npy"), np.stack([st.sumD, st.sumD2]))
        # unique-id broadcast
        uid = qdist.share_unique_id(lambda: bytes(range(128)), rank)
        assert uid == bytes(range(128))
        # max over ranks
        assert qdist.max_over_ranks(float(rank + 1)) == float(world)
        # exchange choice of bench.py at N > 1: every rank must agree
        assert qdist.all_ranks(True) is True
        assert qdist.all_ranks(rank == 0) is False          # one rank's failed attach / self-check
        fused_ms = qdist.max_over_ranks(1.0 + rank)           # the probe times are maxima over ranks
        nccl_ms = qdist.max_over_ranks(1.5)
        assert qdist.pick_exchange(fused_ms, nccl_ms) == "nccl"
        assert qdist.pick_exchange(1.0, 1.5) == "fused"
        # shards tile [0, S)
        cover = torch.zeros(S, dtype=torch.int64)
        cover[off:off + S_l] = 1
        dist.all_reduce(cover)
        assert (cover == 1).all()
    finally:
        dist.destroy_process_group()


def test_sharded_statistics_allreduce_is_exact(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ref = np.load(tmp_path / "ref.npy")
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"sums_{r}.npy"), ref)


def test_shard_validation():
    from paper_2409_02135_b200 import dist as qdist
    assert qdist.shard(64, 8, 3) == (24, 8)
    assert qdist.shard(64, 1, 0) == (0, 64)
    with pytest.raises(ValueError):
        qdist.shard(100, 8, 0)
    with pytest.raises(ValueError):
        qdist.shard(64, 2, 2)


def test_sharded_finalize_matches_unsharded():
    """mu / STD from the all-reduced sums equal the unsharded ones for every shard count."""
    g = gen.random_regular(120, 3, 1)
    st = oracle.run(g, oracle.make_cfg("maxcut", S=48, seed=2), oracle.schedule(-5.0, 0.1, 50)[:9])
    for world in (1, 2, 3, 4, 6, 8):
        parts = [_fixed_point_sums(st.p[:, r * 48 // world:(r + 1) * 48 // world], st.c) for r in range(world)]
        D = sum(p[0] for p in parts)
        D2 = sum(p[1] for p in parts)
        assert np.array_equal(D, st.sumD) and np.array_equal(D2, st.sumD2)
        for i in (0, 7, 119):
            assert oracle.finalize(float(st.c[i]), int(D[i]), int(D2[i]), 48) == \
                oracle.finalize(float(st.c[i]), int(st.sumD[i]), int(st.sumD2[i]), 48)
