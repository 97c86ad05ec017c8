"""Random-order greedy MIS density on a workload graph (context for solution quality; not a pin).
PAPER.md Table 2 reports GREEDY at ApR 0.717 (d=20) / 0.664-0.667 (d=100) against the
asymptotic MIS density, so rho_greedy / ApR_greedy estimates that reference density on our graph."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import gen  # noqa: E402


def greedy_density(g, seed):
    order = np.random.default_rng(seed).permutation(g.n)
    blocked = np.zeros(g.n, bool)
    size = 0
    rp, ci = g.rowptr, g.colidx
    for v in order:
        if not blocked[v]:
            size += 1
            blocked[v] = True
            blocked[ci[rp[v]:rp[v + 1]]] = True
    return size / g.n


if __name__ == "__main__":
    w = gen.workload(sys.argv[1] if len(sys.argv) > 1 else "c5")
    g = w.graphs[0]
    d = [greedy_density(g, s) for s in range(3)]
    print(f"{w.name}: N={g.n} greedy MIS density {np.mean(d):.5f} (seeds 0-2: {', '.join(f'{x:.5f}' for x in d)})")
