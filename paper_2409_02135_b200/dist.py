"""Multi-GPU plumbing around the C ABI (host logic only; the exchange itself is
the library's per-step NCCL all-reduce of the 2n int64 replica-statistic sums).

Replicas are sharded across ranks: rank r holds global replicas
[r*S/G, (r+1)*S/G) of all variables. torch.distributed is used only to share
the 128-byte NCCL unique id and for barriers / max-over-ranks timing.
"""
from __future__ import annotations


def shard(S_total: int, world: int, rank: int) -> tuple[int, int]:
    """(replica_offset, S_local) of ``rank``; the library requires equal shards."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if S_total % world:
        raise ValueError(f"S_total={S_total} is not divisible by {world} ranks")
    S_local = S_total // world
    return rank * S_local, S_local


def share_unique_id(make_id, rank: int, group=None) -> bytes:
    """Rank 0 calls ``make_id()`` (e.g. Solver.nccl_unique_id); every rank returns its bytes."""
    import torch.distributed as dist

    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("unique id must be 128 bytes")
    return bytes(uid)


def attach(solver, rank: int, world: int, group=None) -> None:
    """Collective: give ``solver`` its NCCL communicator over ``world`` ranks."""
    uid = share_unique_id(solver.nccl_unique_id, rank, group)
    solver.attach_comm(uid, rank, world)


def attach_exchange(solver, rank: int, world: int, group=None, mode: str = "atomic"):
    """Collective: the fused statistics exchange over peer memory. Every rank's
    exchange buffer comes from torch symmetric memory, whose rendezvous maps all of them into every
    process; the library gets the peer pointers. Call after ``attach`` (the communicator stays in use
    for init and evaluation). Returns the peer pointers (the buffer is kept alive by ``solver``; another
    handle of the same shape may re-attach to them once ``solver`` is idle)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    nbytes = solver.exchange_bytes()
    grp = group if group is not None else dist.group.WORLD
    try:
        buf = symm.empty(nbytes, dtype=torch.uint8, device=solver.device)
        ok = True
    except Exception:
        buf, ok = None, False
    # agree before the (collective) rendezvous: a rank that could not allocate must not leave the
    # others waiting in it
    if not all_ranks(ok, device=solver.device, group=group):
        raise RuntimeError("symmetric memory unavailable on at least one rank")
    hdl = symm.rendezvous(buf, grp)
    ptrs = list(hdl.buffer_ptrs)
    if len(ptrs) != world or ptrs[rank] != buf.data_ptr():
        raise RuntimeError("symmetric-memory rendezvous returned an unexpected peer map")
    solver.attach_exchange(ptrs, rank, world, keep=(buf, hdl), mode=mode)
    return ptrs


def all_ranks(flag: bool, device=None, group=None) -> bool:
    """True iff ``flag`` holds on every rank (MIN all-reduce): how the ranks agree on using the fused
    exchange (every rank attached it, and its self-check was bit-exact everywhere)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return bool(flag)
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(int(t.item()))


def pick_exchange(fused_ms: float, nccl_ms: float) -> str:
    """'fused' unless the NCCL path was faster; both times are already maxima over ranks, so every rank
    picks the same."""
    return "nccl" if nccl_ms < fused_ms else "fused"


def max_over_ranks(x: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
