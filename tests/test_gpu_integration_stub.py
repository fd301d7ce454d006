"""The ctypes binding INTEGRATION.md tells a manigraph maintainer to add, run
verbatim: the ```python block is extracted from INTEGRATION.md and executed,
then ``embed_b200`` (mg_embed_host: host arrays in, host arrays out) is
compared with ``paper_2112_07862_b200.embed`` and with the reference goldens.
"""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, graph_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stub():
    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import _native
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    block = re.search(r"```python\n(import ctypes as C.*?)```", text, re.S).group(1)
    os.environ["MGB200_LIB"] = _native.LIB_PATH
    ns = {"DisconnectedGraphError": mg.DisconnectedGraphError,
          "ConvergenceError": mg.ConvergenceError, "InputError": mg.InputError}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns


@pytest.mark.parametrize("name,k", [("path10", 2), ("rand3", 3), ("rand700", 4)])
def test_embed_host_matches_embed(stub, golden_small, name, k):
    import paper_2112_07862_b200 as mg
    z, meta = golden_small
    n, ptr, idx, w = graph_from_golden(z, name)
    g = mg.Graph(n, ptr, idx, w)
    cfg = mg.SolverConfig(k=k + 1, tol=1e-8, max_iter=500, seed=42)
    P, ev, b, d = stub["embed_b200"](g, k, cfg)
    emb = mg.embed(g, k, cfg, require_convergence=False)
    # same library, same stream, same order of operations: bit-identical
    assert np.array_equal(P, emb.P)
    assert np.array_equal(ev, emb.eigenvalues)
    assert np.array_equal(b, emb.b)
    assert d.epsilon == emb.diagnostics["epsilon"] and d.mu == emb.diagnostics["mu"]
    assert d.iterations == emb.diagnostics["iterations"]
    key = f"{name}/embed{k}"
    if key in meta:
        ref = z[f"{key}/eigenvalues"]
        assert np.max(np.abs(ev - ref) / np.abs(ref)) < 1e-8


def test_embed_host_errors(stub, golden_small):
    import paper_2112_07862_b200 as mg
    z, _ = golden_small
    g = mg.Graph(*graph_from_golden(z, "twocomp"))
    with pytest.raises(mg.DisconnectedGraphError) as e:
        stub["embed_b200"](g, 1, mg.SolverConfig(k=2))
    assert e.value.n_components == 2
    from paper_2112_07862_b200 import synthetic
    g = mg.Graph(*synthetic.random_connected(np.random.default_rng(5), 150, weighted=True))
    with pytest.raises(mg.ConvergenceError):
        stub["embed_b200"](g, 3, mg.SolverConfig(k=4, tol=1e-12, max_iter=3))


def test_embed_host_reserved_returns_all_pairs(golden_small):
    """cfg.reserved == 1: P and eigenvalues carry all K+1 pairs (the
    host entry point used to size its device P for K columns only)."""
    import ctypes as C
    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import _native as N
    z, meta = golden_small
    n, ptr, idx, w = graph_from_golden(z, "rand3")
    k, m = 3, 4
    lib = N.load()
    ctx = N.context(0)
    zz = np.random.default_rng(42).standard_normal(n * 64 + 8 * n)
    P = np.full((n, m), np.nan)
    b = np.empty(n)
    ev, rn, cv = np.empty(m), np.empty(m), np.empty(m, np.int32)
    hist = np.empty(502)
    out = N.SolverOut()
    out.eigenvalues = ev.ctypes.data_as(N.P_f64)
    out.residual_norms = rn.ctypes.data_as(N.P_f64)
    out.converged = cv.ctypes.data_as(N.P_i32)
    out.history = hist.ctypes.data_as(N.P_f64)
    out.history_cap = hist.size
    s = N.SolverCfg()
    s.k, s.max_iter, s.tol, s.preconditioner, s.precision, s.reorder, s.reserved = m, 500, 1e-8, 1, 0, 1, 1
    dg = N.EmbedDiag()
    ptr = np.ascontiguousarray(ptr, np.int64)
    idx = np.ascontiguousarray(idx, np.int64)
    w = np.ascontiguousarray(w, np.float64)
    N.call("mg_embed_host", ctx, n, ptr.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p),
           w.ctypes.data_as(C.c_void_p), k, C.byref(s), 0, 0, 1, zz.ctypes.data_as(C.c_void_p),
           zz.size, P.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), C.byref(out),
           C.byref(dg))
    assert np.all(np.isfinite(P))
    emb = mg.embed(mg.Graph(n, ptr, idx, w), k, mg.SolverConfig(k=m, tol=1e-8, max_iter=500),
                   require_convergence=False)
    assert np.array_equal(P[:, 1:], emb.P)
    assert np.array_equal(ev[1:], emb.eigenvalues)
    assert ev[0] == emb.diagnostics["dropped_eigenvalue"]
