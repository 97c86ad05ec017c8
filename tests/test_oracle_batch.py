"""NEXT-3 pins (CPU): a batch of instances is the block-diagonal union of their graphs
("batch parallel computation for multiple initial values and instances"), so
  * per-instance evaluation of the union equals evaluating each instance on its own,
  * the counts summed over instances equal the ungrouped evaluation of the union,
  * the annealing dynamics of the union equal independent runs of the instances started
    from the same rows of state (no coupling across instances: the gather stays inside a
    block, the replica statistics are per variable),
  * max clique batches use the union of per-instance complements."""
import numpy as np
import pytest

import gen
import oracle
from oracle import definition as D


def _batch(k=4, problem="mis"):
    if problem == "maxclique":
        gs = [gen.erdos_renyi(20 + 3 * j, 0.6, 300 + j) for j in range(k)]
    else:
        gs = [gen.erdos_renyi(40 + 7 * j, 0.15, 100 + j) for j in range(k)]
    U, gor = gen.disjoint_union(gs)
    return gs, U, gor


def test_disjoint_union_structure():
    gs, U, gor = _batch(5)
    assert U.n == sum(g.n for g in gs) and U.nnz == sum(g.nnz for g in gs)
    u, v = U.edges()
    assert (gor[u] == gor[v]).all()                       # no edge leaves an instance
    assert (np.diff(gor) >= 0).all() and np.array_equal(np.bincount(gor), [g.n for g in gs])
    for k, (a, b) in enumerate(oracle.instance_rows(gor)):
        sub = oracle.subgraph(U, a, b)
        assert np.array_equal(sub.rowptr, gs[k].rowptr) and np.array_equal(sub.colidx, gs[k].colidx)


@pytest.mark.parametrize("problem", ["mis", "maxcut", "maxclique"])
@pytest.mark.parametrize("mp", ["sigmoid", "clamp"])
def test_group_eval_equals_per_instance_eval(problem, mp):
    gs, U, gor = _batch(4, problem)
    rng = np.random.default_rng(1)
    S = 37
    theta = rng.normal(0.5 if mp == "clamp" else 0.0, 1.0, (U.n, S)).astype(np.float32)
    counts, energy, best = oracle.evaluate_groups(U, problem, 2.0, theta, gor, len(gs), map=mp)
    for k, (a, b) in enumerate(oracle.instance_rows(gor)):
        c1, e1, b1 = oracle.evaluate(gs[k], problem, 2.0, theta[a:b], map=mp)
        assert np.array_equal(counts[k], c1) and np.array_equal(energy[k], e1) and best[k] == b1
    if problem != "maxclique":     # the ungrouped union evaluation is the sum over instances
        cu, eu, bu = oracle.evaluate(U, problem, 2.0, theta, map=mp)
        assert np.array_equal(counts.sum(axis=0), cu)


def test_group_complement_is_union_of_complements():
    gs, U, gor = _batch(3, "maxclique")
    rp, ci = oracle.complement_groups(U, gor)
    A = D.dense_adjacency(U.n, rp, ci)
    for k, (a, b) in enumerate(oracle.instance_rows(gor)):
        Ak = D.dense_adjacency(gs[k].n, gs[k].rowptr, gs[k].colidx)
        assert np.array_equal(A[a:b, a:b], D.complement_adjacency(Ak))
        A[a:b, a:b] = 0
    assert not A.any()                                      # nothing between instances


@pytest.mark.parametrize("problem,mp", [("mis", "sigmoid"), ("maxcut", "clamp"), ("maxclique", "sigmoid")])
def test_union_dynamics_equal_independent_instances(problem, mp):
    gs, U, gor = _batch(3, problem)
    S = 24
    cfg = oracle.make_cfg(problem, S=S, seed=7, map=mp, comm=0.3)
    gam = oracle.schedule(-5.0 if problem == "maxcut" else -2.0, 0.1, 200)[:60]
    csr = oracle.complement_groups(U, gor) if problem == "maxclique" else None
    st0 = oracle.init(U, cfg)
    su = oracle.run(U, cfg, gam, state=st0.copy(), csr=csr)
    for k, (a, b) in enumerate(oracle.instance_rows(gor)):
        part = oracle.State(*(getattr(st0, f)[a:b].copy() for f in ("theta", "m", "v", "p", "c", "sumD", "sumD2")), 0)
        sk = oracle.run(gs[k], cfg, gam, state=part)
        for f in ("theta", "m", "v", "p", "c", "sumD", "sumD2"):
            assert np.array_equal(getattr(sk, f), getattr(su, f)[a:b]), (k, f)
