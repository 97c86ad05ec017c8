"""Host-side sizing of the segmented gather (QQA_SEGMENTS) -- no GPU needed.

qqa_workspace_bytes plans the segment CSRs: [KS][n+1] row offsets plus, for every (row, segment), the row's
neighbours in source segment k = [floor(k n / KS), floor((k+1) n / KS)) padded to a multiple of 4. The
workspace growth is checked against that count computed here from the graph, and the shapes the segmented
kernels do not cover keep KS = 1 (no growth)."""
import numpy as np
import pytest

import gen

ALIGN = 256


@pytest.fixture(scope="module")
def Q():
    import paper_2409_02135_b200 as Q
    return Q


def _up(x):
    return (x + ALIGN - 1) // ALIGN * ALIGN


def _seg_entries(g, KS):
    lo = [g.n * k // KS for k in range(KS + 1)]
    seg = np.searchsorted(np.asarray(lo[1:-1]), g.colidx, side="right")    # segment of every column
    row = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    cnt = np.zeros((g.n, KS), np.int64)
    np.add.at(cnt, (row, seg), 1)
    return int(((cnt + 3) // 4 * 4).sum())


@pytest.mark.parametrize("KS", [2, 3, 7])
@pytest.mark.parametrize("mk,S", [(lambda: gen.random_regular(2000, 20, 5), 64),
                                  (lambda: gen.erdos_renyi(900, 0.01, 3), 16),
                                  (lambda: gen.random_regular(1000, 5, 6), 256)])
def test_segment_csr_planned_size(Q, monkeypatch, KS, mk, S):
    g = mk()
    cfg = Q.make_config("mis", S_total=S)
    monkeypatch.delenv("QQA_SEGMENTS", raising=False)
    base = Q.workspace_bytes(g.rowptr, g.colidx, cfg)
    monkeypatch.setenv("QQA_SEGMENTS", str(KS))
    seg = Q.workspace_bytes(g.rowptr, g.colidx, cfg)
    # (the one-pass layout reserves one aligned unit for each of the two empty sections)
    want = _up(KS * (g.n + 1) * 4) + _up(_seg_entries(g, KS) * 4) - 2 * ALIGN
    assert seg - base == want


def test_segments_not_planned_where_unsupported(Q, monkeypatch):
    """VPL > 1 shapes, K-ary colouring and the dense clique keep the one-pass kernel: no segment CSRs."""
    g = gen.random_regular(400, 6, 2)
    for problem, S, extra in [("mis", 512, {}), ("coloring", 16, {"n_colors": 4}), ("maxclique", 16, {})]:
        cfg = Q.make_config(problem, S_total=S, **extra)
        monkeypatch.delenv("QQA_SEGMENTS", raising=False)
        base = Q.workspace_bytes(g.rowptr, g.colidx, cfg)
        monkeypatch.setenv("QQA_SEGMENTS", "4")
        assert Q.workspace_bytes(g.rowptr, g.colidx, cfg) == base, problem
