#!/usr/bin/env python3
"""Ablation workloads of PAPER.md §5.6 (Fig. 3) on the GPU path:

  left    annealing speed: T in {100, 300, 1000, 3000} steps, gamma_0 = -2, sigmoid and clamp maps, on the c4 graph
          (ER-[9000-11000] stand-in, "the largest ER graph")
  middle  initial gamma_0 in {-4, -2, -1, -0.5, 0} at T = 1000, same graph
  right   communication strength alpha_c in {0, 0.1, 0.3, 0.5, 1} with S = 1000 on the c2 batch
          (16 ER-[700-800] stand-ins in one block-diagonal handle, "small ERGs")

Reports the best independent-set size (feasible best replica) averaged over seeds / instances.
Figure 3's values are not in the text, so this is context, not a pin.

  python tools/ablation.py [--out profiles/r1_ablation.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402


def best_size(sol, batched):
    if batched:
        r = sol.round_evaluate_groups(want_x=False)
        sizes = []
        for g in range(r.counts.shape[0]):
            feas = r.counts[g, :, 1] == 0
            sizes.append(int(r.counts[g, feas, 0].max()) if feas.any() else 0)
        return float(np.mean(sizes))
    r = sol.round_evaluate(want_x=False)
    pr = r.per_replica
    feas = pr["violations"] == 0
    return float(pr["size"][feas].max()) if feas.any() else 0.0


def run(g, gor, S, seed, T, gmin, comm, mp="sigmoid"):
    cfg = Q.make_config("mis", S_total=S, seed=seed, comm=comm, map=mp)
    sol = Q.Solver(g.rowptr, g.colidx, cfg, group_of_row=gor)
    t0 = time.perf_counter()
    sol.run_linear(gmin, 0.1, T)
    size = best_size(sol, gor is not None)
    dt = time.perf_counter() - t0
    sol.close()
    return size, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_ablation.json"))
    ap.add_argument("--seeds", type=int, default=3)
    a = ap.parse_args()
    out = {"source": "tools/ablation.py; PAPER.md Fig. 3 (P:479-503) settings on synthetic stand-ins",
           "metric": "best feasible independent-set size (mean over seeds / instances)"}
    w4 = gen.workload("c4")
    g4 = w4.graphs[0]
    rows = []
    for mp in ("sigmoid", "clamp"):
        for T in (100, 300, 1000, 3000):
            r = [run(g4, None, 100, 4000 + s, T, -2.0, 0.1, mp) for s in range(a.seeds)]
            rows.append({"map": mp, "steps": T, "size": float(np.mean([x[0] for x in r])),
                         "seconds": float(np.mean([x[1] for x in r]))})
            print("speed", rows[-1], flush=True)
    out["annealing_speed_c4_S100"] = rows
    rows = []
    for gmin in (-4.0, -2.0, -1.0, -0.5, 0.0):
        r = [run(g4, None, 100, 4000 + s, 1000, gmin, 0.1) for s in range(a.seeds)]
        rows.append({"gamma0": gmin, "size": float(np.mean([x[0] for x in r]))})
        print("gamma0", rows[-1], flush=True)
    out["initial_gamma_c4_S100_T1000"] = rows
    w2 = gen.workload("c2")
    U, gor = w2.batched()
    rows = []
    for comm in (0.0, 0.1, 0.3, 0.5, 1.0):
        size, dt = run(U, gor, 1000, 2000, 3000, -2.0, comm)
        rows.append({"alpha_c": comm, "size": size, "seconds": dt})
        print("comm", rows[-1], flush=True)
    out["communication_c2_S1000_T3000"] = rows
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
