import os, sys, time
sys.path.insert(0, ".")
import gen, paper_2409_02135_b200 as Q
for (r, c, K) in [(5, 5, 5), (6, 6, 7), (7, 7, 7), (8, 8, 9), (9, 9, 10), (8, 12, 12), (11, 11, 11), (13, 13, 13)]:
    g = gen.queens(r, c)
    best = None
    for steps, lr, alpha, gmax, T in [(3000, 0.01, 2, 0.1, 0.0), (30000, 0.01, 4, 1.0, 0.001), (30000, 0.01, 2, 1.0, 0.001)]:
        s = Q.Solver(g.rowptr, g.colidx, Q.make_config("coloring", S_total=1000, seed=1, n_colors=K, lr=lr, alpha=alpha, temperature=T))
        s.run_linear(-2.0, gmax, steps)
        e = int(s.round_evaluate().best_energy)
        best = e if best is None else min(best, e)
        print(f"queen{r}-{c} K={K} steps={steps} lr={lr} a={alpha} gmax={gmax} T={T}: {e}", flush=True)
        s.close()
    print(f"queen{r}-{c}: best {best}", flush=True)
