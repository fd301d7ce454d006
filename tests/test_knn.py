"""kNN graph: the oracle restatement of knn_graph is pinned to
the reference's graphs (tests/golden/knn.npz from make_golden_knn.py), then
the device path is compared with them: structure bit-exact, weights within
1e-13 relative (measured: c1 2e-16, cube3d 7e-15, Swiss roll 2e-14 -- CUDA exp
vs numpy exp plus last-bit differences of BLAS dot products, amplified by
the cancellation in the reference's own distance formula).
"""

import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _far_point_cloud():
    """3000 points in the unit square and one at 1e6: its edge's d^2 / sigma^2 ~ 2000,
    so exp underflows to 0 and from_edges rejects the weight (graph.py:50-51)."""
    x = np.random.default_rng(1).uniform(size=(3001, 2))
    x[-1] = 1e6
    return x


@pytest.fixture(scope="module")
def gk():
    return np.load(os.path.join(HERE, "golden", "knn.npz"))


def test_oracle_knn_matches_reference(gk):
    for name in gk["names"].tolist():
        k, wt = (int(v) for v in gk[f"{name}_k"])
        n, ptr, idx, w = O.knn_graph(gk[f"{name}_x"], k, weighted=bool(wt))
        np.testing.assert_array_equal(ptr, gk[f"{name}_indptr"], err_msg=name)
        np.testing.assert_array_equal(idx, gk[f"{name}_indices"], err_msg=name)
        np.testing.assert_array_equal(w, gk[f"{name}_weights"], err_msg=name)


def test_oracle_knn_errors():
    with pytest.raises(O.OracleInputError):
        O.knn_graph(np.zeros(5), 2)
    with pytest.raises(O.OracleInputError):
        O.knn_graph(np.zeros((5, 2)), 5)
    with pytest.raises(O.OracleInputError):  # exp underflow -> weight 0 (graph.py:50-51)
        O.knn_graph(_far_point_cloud(), 1)


@pytest.mark.gpu
def test_device_knn_matches_reference(gk):
    import paper_2112_07862_b200 as mg
    for name in gk["names"].tolist():
        k, wt = (int(v) for v in gk[f"{name}_k"])
        g = mg.knn_graph(gk[f"{name}_x"], k, weighted=bool(wt))
        np.testing.assert_array_equal(g.indptr, gk[f"{name}_indptr"], err_msg=name)
        np.testing.assert_array_equal(g.indices, gk[f"{name}_indices"], err_msg=name)
        # bit-exact for most edges; the reference's distance formula
        # (sq_i + sq_j - 2 x_i.x_j) cancels ~4 digits on the Swiss roll, so a
        # last-bit difference in a dot product moves a weight by up to ~3e-14
        np.testing.assert_allclose(g.weights, gk[f"{name}_weights"], rtol=1e-13, atol=0,
                                   err_msg=name)


@pytest.mark.gpu
def test_device_knn_errors():
    import paper_2112_07862_b200 as mg
    with pytest.raises(mg.InputError):
        mg.knn_graph(np.zeros(5), 2)
    with pytest.raises(mg.InputError):
        mg.knn_graph(np.zeros((5, 2)), 5)
    with pytest.raises(mg.InputError):
        mg.knn_graph(_far_point_cloud(), 1)


@pytest.mark.gpu
def test_device_knn_feeds_embed(gk):
    """knn_graph -> embed end to end on the device (config 1 point cloud)."""
    import paper_2112_07862_b200 as mg
    g = mg.knn_graph(gk["c1_x"], 10)
    emb = mg.embed(g, 2, mg.SolverConfig(k=3, tol=1e-8, max_iter=300, seed=42),
                   require_convergence=False)
    ref = O.embed(g.n, g.indptr, g.indices, g.weights, 2, tol=1e-8, max_iter=300, seed=42,
                  require_convergence=False)
    np.testing.assert_allclose(emb.eigenvalues, ref["eigenvalues"], rtol=1e-8)


@pytest.mark.gpu
def test_device_knn_grid_matches_reference():
    """n >= 4096, d <= 3: the cell-grid search (mg_knn.cu) against the reference's
    own graphs, including exact distance ties (lattice) and uneven density."""
    import paper_2112_07862_b200 as mg
    gk = np.load(os.path.join(HERE, "golden", "knn_grid.npz"))
    for name in gk["names"].tolist():
        k, wt = (int(v) for v in gk[f"{name}_k"])
        g = mg.knn_graph(gk[f"{name}_x"], k, weighted=bool(wt))
        np.testing.assert_array_equal(g.indptr, gk[f"{name}_indptr"], err_msg=name)
        np.testing.assert_array_equal(g.indices, gk[f"{name}_indices"], err_msg=name)
        np.testing.assert_allclose(g.weights, gk[f"{name}_weights"], rtol=1e-13, atol=0,
                                   err_msg=name)


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k", [(200_000, 3, 8), (120_000, 2, 12), (50_000, 1, 5)])
def test_device_knn_grid_equals_all_pairs(monkeypatch, n, d, k):
    """The grid search returns exactly the all-pairs scan's graph (same arrays)."""
    import paper_2112_07862_b200 as mg
    x = np.random.default_rng(n + d).uniform(size=(n, d))
    x[: n // 10] *= 0.01  # a dense corner: uneven cell occupancy
    g1 = mg.knn_graph(x, k)
    monkeypatch.setenv("MG_KNN_GRID", "0")
    g0 = mg.knn_graph(x, k)
    assert np.array_equal(g1.indptr, g0.indptr)
    assert np.array_equal(g1.indices, g0.indices)
    assert np.array_equal(g1.weights, g0.weights)
