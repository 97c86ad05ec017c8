"""bench.py's exchange selection at N > 1 (select_exchange) on the CPU with world size 2 (gloo): whatever phase
fails on ONE rank -- symmetric-memory attach, the NCCL reference handle, the bit-exact self-check, the timing
probe -- every rank ends on the NCCL handle, none is left waiting in a collective, and with no failure the
faster exchange is kept on both ranks (VERDICT r1 'What's weak' #1). The solver is a stand-in with
the methods the selection calls; the collectives (agreement, max over ranks) are the real ones."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeSolver:
    """The Solver methods select_exchange uses; `fail` names the method that raises on this rank, `bad` makes
    the fused handle's state differ from the reference (a failed self-check)."""

    def __init__(self, kind, fail=None, bad=False):
        self.kind, self.fail, self.bad, self.closed = kind, fail, bad, False

    def _maybe(self, name):
        if self.fail == name:
            raise RuntimeError(f"injected failure in {self.kind}.{name}")

    def reset(self):
        self._maybe("reset")

    def run_linear(self, *a):
        self._maybe("run_linear")

    def get_state(self):
        self._maybe("get_state")
        x = np.zeros((4, 2), np.float32) + (1.0 if (self.bad and self.kind == "fused") else 0.0)
        return {k: x for k in ("theta", "m", "v", "p")}

    def get_stats(self):
        return {"sumD2": np.zeros(4, np.int64)}

    def share_comm(self, donor):
        self._maybe("share_comm")

    def attach_exchange(self, ptrs, rank, world, keep=None, mode="atomic"):
        self._maybe("attach_exchange")
        self.kind, self._exchange_keep, self._exchange_mode = "fused", keep, mode

    def detach_exchange(self):
        self.kind = "nccl"

    def close(self):
        self.closed = True


class FakeEvent:
    def __init__(self, ms):
        self.ms = ms

    def record(self, stream=None):
        pass

    def synchronize(self):
        pass

    def elapsed_time(self, other):
        return other.ms


def _worker(rank, world, port, scenario, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    from paper_2409_02135_b200 import dist as qdist

    fail_rank = 1
    inject = scenario["inject"] if rank == fail_rank else None
    made = []

    def make_solver():
        if inject == "make_solver" and made:   # the reference handle (the second solver made) fails
            raise RuntimeError("injected failure creating the reference handle")
        s = FakeSolver("nccl" if made else "fused", fail=inject if made else None,
                       bad=scenario.get("bad") and rank == 0)
        made.append(s)
        return s

    class QD:   # qdist with the symmetric-memory attach replaced
        all_ranks = staticmethod(qdist.all_ranks)
        pick_exchange = staticmethod(qdist.pick_exchange)

        @staticmethod
        def attach_exchange(sol, r, wsz, mode="atomic"):
            if inject == "attach_exchange":
                raise RuntimeError("injected: no symmetric memory")
            sol._exchange_keep, sol._exchange_mode = None, mode
            return [1, 2]

        @staticmethod
        def attach(sol, r, wsz):
            pass

    fused_ms = scenario.get("fused_ms", 1.0)
    # (start, end) events of the NCCL probe, then of the atomic and the slotted fused probes
    seq = iter([0.0, 2.0, 0.0, fused_ms, 0.0, scenario.get("slotted_ms", fused_ms)])
    bench.torch_event = lambda: FakeEvent(next(seq))
    args = type("A", (), {"exchange": "auto"})()
    w = type("W", (), {"n_colors": 0, "gamma_min": -2.0, "gamma_max": 0.1, "steps": 10})()
    sol = make_solver()
    res = bench.select_exchange(args, w, None, QD, sol, make_solver, rank, world, None, None,
                                lambda: dist.barrier(), lambda x: qdist.max_over_ranks(x))
    kept, xptrs, desc, probe = res
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"kind": kept.kind, "fused": xptrs is not None, "desc": desc,
                   "mode": getattr(kept, "_exchange_mode", None)}, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("scenario", [
    {"inject": "attach_exchange", "expect": "nccl"},
    {"inject": "make_solver", "expect": "nccl"},
    {"inject": "run_linear", "expect": "nccl"},      # raises inside the self-check on one rank
    {"inject": None, "bad": True, "expect": "nccl"},  # rank 0's fused state differs: self-check fails
    {"inject": "reset", "expect": "nccl"},           # the reference handle's reset raises in the self-check
    {"inject": "get_state", "expect": "nccl"},       # the reference handle's state read raises
    {"inject": None, "fused_ms": 1.0, "expect": "fused"},
    {"inject": None, "fused_ms": 3.0, "expect": "nccl"},
    {"inject": None, "fused_ms": 3.0, "slotted_ms": 1.5, "expect": "fused", "mode": "slotted"},
    {"inject": None, "fused_ms": 1.2, "slotted_ms": 1.5, "expect": "fused", "mode": "atomic"},
])
def test_every_rank_agrees_on_the_exchange(tmp_path, scenario):
    mp.start_processes(_worker, args=(2, _free_port(), scenario, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    got = [json.load(open(tmp_path / f"r{r}.json")) for r in range(2)]
    assert got[0]["fused"] == got[1]["fused"], got
    assert got[0]["fused"] == (scenario["expect"] == "fused"), got
    if "mode" in scenario:
        assert got[0]["mode"] == got[1]["mode"] == scenario["mode"], got
