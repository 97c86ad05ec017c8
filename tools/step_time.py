#!/usr/bin/env python3
"""Per-step kernel time of one workload (A/B helper): python tools/step_time.py c5 [steps]
Environment variables (QQA_BLOCK_REPLICAS, QQA_PERSISTENT, QQA_CLUSTER, QQA_LIB_PATH, ...) select the variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
w = gen.workload(name)
(g, gor) = w.batched()          # a batch (c2, t1) runs as one block-diagonal handle, as bench.py does
hp = {k: v for k, v in w.hparams().items() if k != "problem"}
sol = Q.Solver(g.rowptr, g.colidx, Q.make_config(w.problem, S_total=w.S, seed=w.seeds[0], **hp), group_of_row=gor)
sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 5)   # warm-up
sol.profile(True)
sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 5, 5 + steps)
ms, k = sol.profile_read()
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("QQA_"))
print(f"{name} path={sol.step_path()} {env or '(default)'}: {1e3 * ms / k:.1f} us/step over {k} steps")
