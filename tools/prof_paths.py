#!/usr/bin/env python3
"""ncu targets for the newer step paths: python tools/prof_paths.py cluster|quad
cluster: c1 on k_run_cluster (one launch of 200 steps); quad: q13 on k_step_Kq (10 steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cluster"
w = gen.workload("c1" if which == "cluster" else "q13")
g = w.graphs[0]
hp = {k: v for k, v in w.hparams().items() if k != "problem"}
sol = Q.Solver(g.rowptr, g.colidx, Q.make_config(w.problem, S_total=w.S, seed=w.seeds[0], **hp))
sol.run_linear(w.gamma_min, w.gamma_max, w.steps, 0, 200 if which == "cluster" else 10)
print(which, sol.step_path(), sol.get_state()["step"])
