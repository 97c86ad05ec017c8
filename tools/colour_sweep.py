#!/usr/bin/env python3
"""Solution-quality sweep of K-ary PQQA on queen13-13 (K = 13, S = 1000): best conflicts per setting.
Context for DESIGN.md §9 (the paper's Table 4 reports 14 conflicts; its colouring hyper-parameters are
not printed). python tools/colour_sweep.py"""
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402

g = gen.queens(13, 13)
print("steps lr alpha gmin gmax T comm -> best conflicts (seconds)")
for steps, lr, alpha, gmin, gmax, T, comm in itertools.product(
        [3000, 30000], [0.01, 0.003], [2, 4], [-2.0], [0.1, 1.0], [0.0, 0.001], [0.1]):
    t = time.time()
    s = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=1000, seed=1, n_colors=13, lr=lr, alpha=alpha,
                                                   temperature=T, comm=comm))
    s.run_linear(gmin, gmax, steps)
    r = s.round_evaluate()
    print(steps, lr, alpha, gmin, gmax, T, comm, "->", int(r.best_energy), f"({time.time() - t:.1f})", flush=True)
    s.close()
