"""GPU parity at BASELINE.json config scale (C1 is in test_gpu_parity.py).

Tolerances are derived from the reference's own rounding noise:
at tol 1e-6 two fp64 runs of the reference that differ by one ulp in A agree
to 3.5e-10 ... 2.2e-8 relative in the eigenvalues and 1.7e-6 ... 8.9e-5 rad
per column, and both sit ~2.4e-7 ... 7.6e-7 from the tight (shift-invert)
eigenvalues.  The north_star's fp32 bars are 1e-4 relative / 1e-3 rad.
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


@pytest.fixture(scope="module")
def c2_graph(golden_c2):
    from paper_2112_07862_b200 import synthetic
    z, meta = golden_c2
    g = synthetic.config_graph("c2")
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(g[1]).tobytes()).hexdigest() == meta["graph"]["sha_indptr"]
    assert hashlib.sha256(np.ascontiguousarray(g[2]).tobytes()).hexdigest() == meta["graph"]["sha_indices"]
    return g


def _embed_full(mg, g, K, cfg, reorder=True):
    from paper_2112_07862_b200 import core
    old = os.environ.get("MG_REORDER")
    os.environ["MG_REORDER"] = "1" if reorder else "0"
    try:
        n, ptr, idx, w = g
        res, b, dg = core.embed_arrays(n, ptr, idx, w, K, cfg)
    finally:
        if old is None:
            del os.environ["MG_REORDER"]
        else:
            os.environ["MG_REORDER"] = old
    return res.eigenvalues, res.eigenvectors.cpu().numpy(), b.cpu().numpy(), dg, res


def test_c2_operator_pair_bit_exact(mg, golden_c2, c2_graph):
    z, meta = golden_c2
    pair = mg.build_operator_pair(mg.Graph(*c2_graph))
    import hashlib
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for key, arr in (("A_ptr", pair.A.indptr), ("A_idx", pair.A.indices), ("Q_ptr", pair.Q.indptr),
                     ("Q_idx", pair.Q.indices), ("Q_val", pair.Q.data)):
        assert sha(arr) == meta["pair"][f"sha_{key}"], key
    # eps: faithful replica of the 60-iteration best-effort Ritz value (F2)
    assert abs(pair.epsilon - meta["pair"]["eps"]) <= 1e-10 * meta["pair"]["eps"]
    assert abs(pair.mu - meta["pair"]["mu"]) <= 1e-10 * meta["pair"]["mu"]
    b = z["b"]
    assert np.max(np.abs(pair.B.b - b) / b) < 1e-9


@pytest.mark.parametrize("reorder", [True, False])
def test_c2_fp64_eigenpairs(mg, golden_c2, c2_graph, reorder):
    z, meta = golden_c2
    cfg = mg.SolverConfig(k=5, tol=1e-6, max_iter=3000, seed=42)
    ev, vecs, b, dg, res = _embed_full(mg, c2_graph, 4, cfg, reorder)
    ref = z["eigenvalues"]
    tight = z["tight_eigenvalues"]
    assert res.converged.all()
    # tol 1e-6 bounds each run's error vs the truth (reference: 2.4e-7..7.6e-7,
    # SURVEY F5), so two valid runs agree to ~2x that; reordering changes every
    # summation order, so the 1-ulp noise band (2.2e-8) does not apply
    assert np.max(np.abs(ev - ref) / ref) < (5e-8 if not reorder else 1e-6)
    assert np.max(np.abs(ev - tight) / tight) < 2e-6      # tol-derived accuracy
    assert abs(dg.epsilon - meta["pair"]["eps"]) <= 1e-10 * meta["pair"]["eps"]
    ang = principal_angles(vecs, z["eigenvectors"].astype(np.float64), b)
    assert ang.max() < 3e-4
    # B-orthonormality of the returned block
    gram = vecs.T @ (b[:, None] * vecs)
    assert np.max(np.abs(gram - np.eye(5))) < 1e-8
    # the reference needs 1001; measured 1001 (reordered) and 998 (natural
    # order): the last pair crosses tol 1e-6 inside the F5 noise band
    assert abs(res.iterations - meta["solve"]["iterations"]) <= 5, res.iterations


def _angles_vs_tight(z, vecs, b):
    tight = z["tight_eigenvectors6"].astype(np.float64)
    ref = z["eigenvectors"].astype(np.float64)
    ours = [float(principal_angles(vecs[:, [j]], tight[:, [j]], b)[0]) for j in range(5)]
    theirs = [float(principal_angles(ref[:, [j]], tight[:, [j]], b)[0]) for j in range(5)]
    return np.array(ours), np.array(theirs)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c2_vectors_vs_tight_solution(mg, golden_c2, c2_graph, precision):
    """Per-column distance to the shift-invert solution is no worse than the
    reference's own (x2.5) or the north_star bar (1e-6 fp64 / 1e-3 fp32).
    At tol 1e-6 the reference's top vector is itself 1.5e-3 rad off (gap 9e-5)."""
    z, meta = golden_c2
    cfg = mg.SolverConfig(k=5, tol=1e-6, max_iter=3000, seed=42, precision=precision)
    ev, vecs, b, dg, res = _embed_full(mg, c2_graph, 4, cfg)
    ours, theirs = _angles_vs_tight(z, vecs, b)
    if precision == "fp64":
        assert np.all(ours <= np.maximum(1e-6, 2.5 * theirs)), (ours, theirs)
        return
    # fp32: north_star bar on every column the reference resolves below it ...
    well = theirs < 1e-3
    assert np.all(ours[well] <= 1e-3), (ours, theirs)
    # ... and the a-posteriori (Davis-Kahan, B inner product) bound everywhere:
    # sin angle_j <= ||A x_j - theta_j B x_j||_{B^-1} / dist(theta_j, other eigenvalues)
    pair = mg.build_operator_pair(mg.Graph(*c2_graph))
    lam = z["tight_eigenvalues6"]
    for j in range(5):
        x = vecs[:, j]
        th = float(x @ pair.A.matvec(x)) / float(x @ (b * x))
        r = pair.A.matvec(x) - th * b * x
        rn = np.sqrt(np.sum(r * r / b)) / np.sqrt(float(x @ (b * x)))
        gap = np.min(np.abs(np.delete(lam, j) - th))
        assert ours[j] <= 1.05 * rn / gap + 1e-6, (j, ours[j], rn / gap)


def test_c2_fp32_eigenpairs(mg, golden_c2, c2_graph):
    z, meta = golden_c2
    cfg = mg.SolverConfig(k=5, tol=1e-6, max_iter=3000, seed=42, precision="fp32")
    ev, vecs, b, dg, res = _embed_full(mg, c2_graph, 4, cfg)
    ref = z["eigenvalues"]
    assert res.converged.all()
    assert np.max(np.abs(ev - ref) / ref) < 1e-4          # north_star fp32 bar
    # difference-form SpMM keeps fp32 eigenvalues near fp64 accuracy
    assert np.max(np.abs(ev - z["tight_eigenvalues"]) / z["tight_eigenvalues"]) < 5e-6
    gram = vecs.T @ (b[:, None] * vecs)
    assert np.max(np.abs(gram - np.eye(5))) < 1e-4


@pytest.mark.slow
def test_c3_sphere_fp32_self_consistent(mg):
    """Config 3 (1M sphere, K=8, fp32): converged, B-orthonormal, small
    residuals measured with an fp64 oracle SpMM, spherical-harmonic clusters."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.config_graph("c3")
    cfg = mg.SolverConfig(k=9, tol=1e-5, max_iter=3000, seed=42, precision="fp32")
    ev, vecs, b, dg, res = _embed_full(mg, g, 8, cfg)
    assert res.converged.all()
    gram = vecs.T @ (b[:, None] * vecs)
    assert np.max(np.abs(gram - np.eye(9))) < 1e-3
    # l = 1 cluster (3-fold) and l = 2 cluster (5-fold) of the sphere
    rel = np.diff(ev) / ev[1:]
    assert rel[1] < 5e-2 and rel[2] < 5e-2        # 3-fold l=1
    assert rel[3] > 5e-2                          # gap to l=2
    # fp64 residuals of the fp32 eigenvectors against the fp64 operator pair
    pair = mg.build_operator_pair(mg.Graph(*g))
    assert abs(pair.epsilon - dg.epsilon) <= 1e-3 * dg.epsilon
    r = pair.A.matmat(vecs) - (b[:, None] * vecs) * ev
    n = g[0]
    anorm = np.sqrt(np.sum(pair.A.data ** 2)) / np.sqrt(n)
    crit = 1e-5 * (anorm + np.abs(ev) * b.max()) * np.linalg.norm(vecs, axis=0)
    assert np.all(np.linalg.norm(r, axis=0) <= 3 * crit)


def _kmeans_labels(x, c, seed=0, iters=100):
    """Plain k-means++ / Lloyd (the reference's clustering.py:57-96 recipe, numpy
    RNG) -- test infrastructure for the C4 label check."""
    rng = np.random.default_rng(seed)
    n = x.shape[0]
    centers = np.empty((c, x.shape[1]))
    centers[0] = x[rng.integers(n)]
    d2 = np.sum((x - centers[0]) ** 2, axis=1)
    for j in range(1, c):
        centers[j] = x[rng.choice(n, p=d2 / d2.sum())]
        d2 = np.minimum(d2, np.sum((x - centers[j]) ** 2, axis=1))
    labels = np.full(n, -1)
    for _ in range(iters):
        d = (x * x).sum(1)[:, None] - 2 * x @ centers.T + (centers * centers).sum(1)[None, :]
        new = np.argmin(d, axis=1)
        if np.array_equal(new, labels):
            break
        labels = new
        for j in range(c):
            if np.any(labels == j):
                centers[j] = x[labels == j].mean(axis=0)
    return labels


def _same_partition(a, b):
    """Labels equal up to a permutation of the label values."""
    pairs = set(zip(a.tolist(), b.tolist()))
    return len(pairs) == len(set(a.tolist())) == len(set(b.tolist()))


@pytest.mark.slow
def test_c4_disconnected_patches_kmeans_labels(mg):
    """Config 4 family (10 disjoint unit squares, kNN k=10, K=16, fp32, tol 1e-5) at
    10 x 20K points: embed() raises DisconnectedGraphError like the reference
    (embedding.py:53-58); the harness path without the check
    converges, and k-means with 10 clusters on the row-normalised indicator
    block recovers the 10 patches exactly (labels identical up to permutation)."""
    from paper_2112_07862_b200 import core, synthetic
    n = 200_000
    g = synthetic.config_graph("c4", n=n)
    truth = np.arange(n) // (n // 10)
    cfg = mg.SolverConfig(k=17, tol=1e-5, max_iter=3000, seed=42, precision="fp32")
    with pytest.raises(mg.DisconnectedGraphError) as ei:
        mg.embed(mg.Graph(*g), 16, cfg)
    assert ei.value.n_components == 10
    res, b, dg = core.embed_arrays(*g, 16, cfg, check_connected=False)
    assert res.converged.all()
    vecs = res.eigenvectors.cpu().numpy()
    bb = b.cpu().numpy()
    gram = vecs.T @ (bb[:, None] * vecs)
    assert np.max(np.abs(gram - np.eye(17))) < 1e-3
    # the 10 smallest pairs span the component indicators (a near-degenerate
    # cluster at ~eps, then a gap): the rotation-invariant readout is k-means on
    # the row-normalised first 10 columns (clustering.normalize_rows, the
    # reference's angular readout), here on the device k-means as well
    ev = res.eigenvalues
    assert (ev[9] - ev[0]) < 1e-2 * ev[0] < (ev[10] - ev[9])
    x10 = mg.normalize_rows(vecs[:, :10])
    assert _same_partition(_kmeans_labels(x10, 10), truth)
    assert _same_partition(mg.kmeans(x10, 10, restarts=4, seed=42), truth)


@pytest.mark.slow
def test_c5_cube_fp32_self_consistent(mg):
    """Config 5 family (uniform unit cube, kNN k=8, K=32, fp32 + fp64 Gram, tol 1e-4)
    at 200K points: converged, B-orthonormal, fp64-checked residuals within 3x the
    reference's convergence test, and the cube's first 3-fold cluster
    (Neumann modes cos(pi x), cos(pi y), cos(pi z)) separated from the next."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.config_graph("c5", n=200_000)
    cfg = mg.SolverConfig(k=33, tol=1e-4, max_iter=3000, seed=42, precision="fp32")
    ev, vecs, b, dg, res = _embed_full(mg, g, 32, cfg)
    assert res.converged.all()
    gram = vecs.T @ (b[:, None] * vecs)
    assert np.max(np.abs(gram - np.eye(33))) < 1e-3
    rel = np.diff(ev) / ev[1:]
    assert rel[1] < 5e-2 and rel[2] < 5e-2       # 3-fold (1,0,0) modes
    assert rel[3] > 1e-1                         # gap to the (1,1,0) cluster
    pair = mg.build_operator_pair(mg.Graph(*g))
    assert abs(pair.epsilon - dg.epsilon) <= 1e-3 * dg.epsilon
    r = pair.A.matmat(vecs) - (b[:, None] * vecs) * ev
    anorm = np.sqrt(np.sum(pair.A.data ** 2)) / np.sqrt(g[0])
    crit = 1e-4 * (anorm + np.abs(ev) * b.max()) * np.linalg.norm(vecs, axis=0)
    assert np.all(np.linalg.norm(r, axis=0) <= 3 * crit)
