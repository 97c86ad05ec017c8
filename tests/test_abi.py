"""C-ABI boundary checks that need no GPU: the library loads, exports every
function include/qqa.h declares, and host-only entry points validate input."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def Q():
    import paper_2409_02135_b200 as Q
    return Q


def test_library_exports_every_header_symbol(Q):
    names = Q.header_functions()
    assert len(names) >= 18
    out = subprocess.check_output(["nm", "-D", "--defined-only", Q.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (qqa_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert getattr(Q.lib, n) is not None


def test_library_is_sm100a(Q):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", Q.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_version_and_status_strings(Q):
    assert Q.lib.qqa_version() == 9
    assert Q.lib.qqa_status_string(2) == b"bad graph"


def _ws(Q, g, cfg):
    return Q.workspace_bytes(g.rowptr, g.colidx, cfg)


def test_workspace_bytes_scales(Q):
    g = gen.random_regular(1000, 4, 1)
    a = _ws(Q, g, Q.make_config("mis", S_total=16))
    b = _ws(Q, g, Q.make_config("mis", S_total=64))
    # five [n][S_p] float arrays dominate
    assert b - a == pytest.approx(5 * 1000 * (64 - 16) * 4, rel=0.05)
    c = _ws(Q, g, Q.make_config("maxclique", S_total=16))
    assert c > a  # complement graph is much denser


@pytest.mark.parametrize("bad,status", [
    (dict(alpha=3), 1), (dict(alpha=0), 1), (dict(beta1=1.0), 1), (dict(comm=-0.1), 1),
    (dict(S_total=0), 1), (dict(S_total=4, S_local=8), 1), (dict(S_total=4096, S_local=2048), 6),
    (dict(problem=7), 1),
])
def test_invalid_config_rejected(Q, bad, status):
    g = gen.random_regular(20, 3, 1)
    kw = dict(problem="mis", S_total=16)
    prob = bad.pop("problem", "mis")
    kw.update(bad)
    kw["problem"] = prob
    with pytest.raises(Q.QQAError) as e:
        _ws(Q, g, Q.make_config(**kw))
    assert e.value.status == status


def test_bad_rowptr_rejected_on_host(Q):
    g = gen.random_regular(20, 3, 1)
    rp = g.rowptr.copy()
    rp[5], rp[6] = rp[6], rp[5]
    with pytest.raises(Q.QQAError) as e:
        Q.workspace_bytes(rp, g.colidx, Q.make_config("mis", S_total=8))
    assert e.value.status == 2


def test_product_path_never_touches_oracle():
    """The CUDA path and its binding share no code with oracle/ and never import it."""
    pkg = os.path.join(ROOT, "paper_2409_02135_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", text.replace("oracle-matching", "")), f


def test_create_without_gpu_fails_cleanly(Q):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = gen.random_regular(20, 3, 1)
    cfg = Q.make_config("mis", S_total=8)
    h = ctypes.c_void_p(0)
    G = Q._lib.Graph(g.n, g.nnz, g.rowptr.ctypes.data, g.colidx.ctypes.data)
    st = Q.lib.qqa_create(ctypes.byref(h), ctypes.byref(G), ctypes.byref(cfg), ctypes.c_void_p(256),
                          ctypes.c_size_t(1 << 30), None)
    assert st in (3, 7)  # CUDA (no device) or WORKSPACE (not device memory)
    assert Q.lib.qqa_last_error()
