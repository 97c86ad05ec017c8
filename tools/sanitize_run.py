#!/usr/bin/env python3
"""Small run through every kernel path of libqqa.so, for compute-sanitizer:
create (validate, pad), init, launch-per-step, persistent and one-cluster steps, blocked layout, clamp /
noise, batches, weights, K-ary colouring, the printed clique relaxation, loopback shards (NCCL-style and
fused exchange), checkpoint / resume and every evaluation kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_02135_b200 as Q  # noqa: E402


def main():
    g = gen.erdos_renyi(300, 0.04, 1)
    gam = np.linspace(-2.0, 0.1, 40, dtype=np.float32)
    for problem, hp in [("mis", {}), ("maxcut", dict(map="clamp", temperature=0.001)), ("maxclique", {}),
                        ("maxclique_sparse", {}), ("mis", dict(alpha=4, comm=0.5))]:
        gg = gen.erdos_renyi(60, 0.5, 2) if problem == "maxclique" else g
        s = Q.Solver(gg.rowptr, gg.colidx, Q.make_config(problem, S_total=37, seed=3, **hp))
        s.run(gam[:1])                     # launch-per-step
        s.run(gam[1:])                     # persistent (if eligible)
        r = s.round_evaluate()
        st = s.get_state()
        s.set_state(st["theta"], st["m"], st["v"], st["step"], c=s.get_stats()["c"])
        s.run(gam[:3])
        s.round_evaluate_groups()
        s.close()
    os.environ["QQA_BLOCK_REPLICAS"] = "8"
    s = Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=45, seed=4, temperature=0.001))
    s.run(gam)
    s.round_evaluate()
    s.close()
    del os.environ["QQA_BLOCK_REPLICAS"]
    U, gor = gen.disjoint_union([gen.erdos_renyi(50, 0.1, k) for k in range(4)])
    s = Q.Solver(U.rowptr, U.colidx, Q.make_config("mis", S_total=20, seed=5), group_of_row=gor)
    s.run(gam)
    s.round_evaluate_groups()
    s.round_evaluate()
    s.close()
    gw = gen.with_weights(g, "pm1", 6)
    s = Q.Solver(gw.rowptr, gw.colidx, Q.make_config("maxcut", S_total=16, seed=6), weights=gw.weights)
    s.run(gam)
    s.round_evaluate()
    s.close()
    q = gen.queens(5, 5)
    for K, S in ((5, 37), (13, 100)):
        s = Q.Solver(q.rowptr, q.colidx, Q.make_config("coloring", S_total=S, seed=7, n_colors=K, lr=0.1,
                                                       temperature=0.001))
        s.run(gam)
        s.round_evaluate()
        st = s.get_state()
        s.set_state(st["theta"], st["m"], st["v"], st["step"])
        s.close()
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config("mis", S_total=24, seed=8, replica_offset=r * 8, S_local=8))
              for r in range(3)]
    Q.loopback_sync_init(shards)
    Q.loopback_run(shards, gam[:10])
    for s in shards:
        s.round_evaluate()
    # fused statistics exchange (k_step_x) on emulated shards, each with its own exchange buffer
    import torch
    shards = [Q.Solver(g.rowptr, g.colidx, Q.make_config("maxcut", S_total=24, seed=9, replica_offset=r * 8, S_local=8,
                                                         temperature=0.001)) for r in range(3)]
    bufs = [torch.empty(sh.exchange_bytes(), dtype=torch.uint8, device=sh.device) for sh in shards]
    for r, sh in enumerate(shards):
        sh.attach_exchange([b.data_ptr() for b in bufs], r, 3, keep=bufs)
    Q.loopback_sync_init(shards)
    Q.loopback_run(shards, gam[:10])
    for s in shards:
        s.get_stats()
        s.round_evaluate()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
