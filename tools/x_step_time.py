#!/usr/bin/env python3
"""Per-step kernel time of the sharded paths at one rank (A/B helper): c5's graph with S_l replicas,
NCCL communicator (k_finalize + k_step) vs the fused exchanges (k_step_x: atomics; k_step_xs: owner slots).
  python tools/x_step_time.py [S_l] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402

S_l = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
w = gen.workload("c5")
g = w.graphs[0]
hp = {k: v for k, v in w.hparams().items() if k != "problem"}
for mode in ("nccl", "fused", "slotted"):
    sol = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=S_l, seed=5, S_local=S_l, **hp))
    sol.attach_comm(Q.Solver.nccl_unique_id(), 0, 1)
    if mode in ("fused", "slotted"):
        buf = torch.empty(sol.exchange_bytes(), dtype=torch.uint8, device=sol.device)
        sol.attach_exchange([buf.data_ptr()], 0, 1, keep=buf, mode="atomic" if mode == "fused" else "slotted")
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 5)
    sol.profile(True)
    sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 5, 5 + steps)
    ms, k = sol.profile_read()
    print(f"S_l={S_l} {mode} path={sol.step_path()}: {1e3 * ms / k:.1f} us per step kernel over {k} steps", flush=True)
    sol.close()
