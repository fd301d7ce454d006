"""Row-partitioned solve on one B200: R virtual ranks as threads
with the host-rendezvous communicator, compared with the single-GPU embed.

The setup is replicated, so Q and the nnz counts are identical; eps and the
eigenpairs come from iterative solves whose reductions are summed in a
different order (per-rank partials, then the allreduce), so they agree to the
solver tolerance, like the reordered single-GPU run (test_gpu_configs), and
mu / A / b inherit eps's last-ulp noise.
"""

import os

import numpy as np
import pytest

from conftest import principal_angles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mg():
    import paper_2112_07862_b200 as mg
    return mg


def _single(g, K, cfg):
    from paper_2112_07862_b200 import core
    n, ptr, idx, w = g
    res, b, dg = core.embed_arrays(n, ptr, idx, w, K, cfg)
    return res, b.cpu().numpy(), dg


def _dist(g, K, cfg, R, reorder=True):
    from paper_2112_07862_b200 import dist
    n, ptr, idx, w = g
    def body(comm, ctx, r):
        res, b, dg = dist.embed_arrays_dist(comm, ctx, 0, n, ptr, idx, w, K, cfg, reorder=reorder)
        res.eigenvectors = res.eigenvectors.cpu().numpy()
        return res, b.cpu().numpy(), dg
    return dist.run_local(R, body)


def _compare(g, K, cfg, R, ev_tol, ang_tol):
    res0, b0, dg0 = _single(g, K, cfg)
    f64 = cfg.precision == "fp64"
    rt = 1e-9 if f64 else 1e-6  # eps / mu / b: inherited from the eps solve
    outs = _dist(g, K, cfg, R)
    assert len(outs) == R
    for r, (res, b, dg) in enumerate(outs):
        assert res.converged.all(), r
        # replicated setup; b inherits eps's reduction-order noise (ulps)
        np.testing.assert_allclose(b, b0, rtol=rt, atol=0)
        assert dg.mu == pytest.approx(dg0.mu, rel=rt)
        assert dg.epsilon == pytest.approx(dg0.epsilon, rel=rt)
        assert dg.q_nnz == dg0.q_nnz and dg.a_nnz == dg0.a_nnz
        ev = res.eigenvalues
        assert np.max(np.abs(ev - res0.eigenvalues) / np.abs(res0.eigenvalues)) < ev_tol
        vecs = res.eigenvectors
        ang = principal_angles(vecs, res0.eigenvectors.cpu().numpy(), b)
        assert ang.max() < ang_tol, ang
        gram = vecs.T @ (b[:, None] * vecs)
        assert np.max(np.abs(gram - np.eye(K + 1))) < (1e-8 if cfg.precision == "fp64" else 1e-4)
    # every rank returns the same full embedding
    for res, b, dg in outs[1:]:
        np.testing.assert_array_equal(res.eigenvalues, outs[0][0].eigenvalues)
        np.testing.assert_array_equal(res.eigenvectors, outs[0][0].eigenvectors)


@pytest.mark.parametrize("R", [2, 3])
def test_dist_small_natural_order(mg, R):
    """n <= 4096: no reordering, large halos (every rank talks to every rank)."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.random_connected(np.random.default_rng(5), 1500, extra=3000, weighted=True)
    cfg = mg.SolverConfig(k=5, tol=1e-8, max_iter=2000, seed=42)
    _compare(g, 4, cfg, R, 1e-9, 1e-5)


@pytest.mark.parametrize("R,precision", [(2, "fp64"), (4, "fp64"), (2, "fp32")])
def test_dist_c2(mg, R, precision):
    """Config 2 graph (100k kNN, Cuthill-McKee order, thin halos)."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.config_graph("c2")
    cfg = mg.SolverConfig(k=5, tol=1e-6, max_iter=3000, seed=42, precision=precision)
    if precision == "fp64":
        _compare(g, 4, cfg, R, 1e-6, 3e-4)
    else:
        _compare(g, 4, cfg, R, 1e-4, 1e-2)


def test_nccl_single_rank_communicator(mg):
    """NCCL is loaded (dlopen), a unique id is made and a 1-rank communicator
    runs the distributed entry point (which then takes the unpartitioned path)."""
    from paper_2112_07862_b200 import _native as N, dist
    import ctypes as C
    uid = dist.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    N.call("mg_comm_create_nccl", N.context(0), 1, 0, C.cast(buf, C.c_void_p), C.byref(h))
    comm = dist.Comm(h, 0, 1, "nccl")
    from paper_2112_07862_b200 import synthetic
    g = mg.Graph(*synthetic.random_connected(np.random.default_rng(2), 600, extra=900,
                                             weighted=True))
    cfg = mg.SolverConfig(k=4, tol=1e-8, max_iter=2000, seed=42)
    e1 = dist.embed_dist(comm, g, 3, cfg)
    e0 = mg.embed(g, 3, cfg)
    np.testing.assert_array_equal(e1.eigenvalues, e0.eigenvalues)
    np.testing.assert_array_equal(e1.P, e0.P)
    comm.close()


def test_dist_c5_block_width_fast_paths(mg):
    """K = 32 (w = 108), fp32: the tensor-core update, the narrow Gram with derived blocks
    and the breakdown guard run under the row partition too (2 virtual ranks); every rank
    ends with the same converged block, Ritz values equal to the single-GPU solve's to the
    stopping rule's resolution."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.config_graph("c5", n=60_000)
    cfg = mg.SolverConfig(k=33, tol=1e-4, max_iter=3000, seed=42, precision="fp32")
    res0, b0, _ = _single(g, 32, cfg)
    outs = _dist(g, 32, cfg, 2)
    for res, b, dg in outs:
        assert res.converged.all()
        rel = np.abs(res.eigenvalues - res0.eigenvalues) / np.abs(res0.eigenvalues)
        assert rel[:26].max() < 3e-3, rel
        vecs = res.eigenvectors
        gram = vecs.T @ (b[:, None] * vecs)
        assert np.max(np.abs(gram - np.eye(33))) < 1e-4
    np.testing.assert_array_equal(outs[0][0].eigenvalues, outs[1][0].eigenvalues)
    np.testing.assert_array_equal(outs[0][0].eigenvectors, outs[1][0].eigenvectors)
