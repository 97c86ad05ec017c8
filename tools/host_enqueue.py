#!/usr/bin/env python3
"""Host enqueue cost of the sharded (NCCL) step path vs its device time.

One process, a one-rank NCCL communicator (the N > 1 code path at N = 1: k_finalize + 4 row-chunk k_step
launches + 4 grouped all-reduces + events per step). Prints host microseconds per step spent inside
qqa_run_linear (enqueue only) and device microseconds per step (CUDA events), for S_local replicas of c5
(S_local = 64 / G stands in for one rank of a G-GPU run).
  python tools/host_enqueue.py [S_local ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402
from paper_2409_02135_b200 import dist as qdist  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
w = gen.workload("c5")
g = w.graphs[0]
hp = {k: v for k, v in w.hparams().items() if k != "problem"}
T = 300
for S_l in [int(x) for x in sys.argv[1:]] or [8, 16, 32, 64]:
    cfg = Q.make_config("mis", S_total=S_l, seed=5, S_local=S_l, **hp)
    sol = Q.Solver(g.rowptr, g.colidx, cfg, device=dev)
    qdist.attach(sol, 0, 1)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sol.stream)
    h0 = time.perf_counter()
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 20, 20 + T)
    h1 = time.perf_counter()
    e1.record(sol.stream)
    torch.cuda.synchronize()
    print(f"S_local={S_l} launches/step={(sol.launch_count()) / (20 + T):.1f}: host enqueue "
          f"{1e6 * (h1 - h0) / T:.1f} us/step, device {1e3 * e0.elapsed_time(e1) / T:.1f} us/step", flush=True)
    sol.close()
dist.destroy_process_group()
