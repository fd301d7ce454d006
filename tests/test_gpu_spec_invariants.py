"""GPU checks of the reference SPEC's LOBPCG / embedding invariants.

SURVEY §4 lists these as "SPEC known answers that are not implemented as tests"
in the reference.  Each is exercised here through
the sm_100a path (``lobpcg_smallest`` / ``embed`` / ``fiedler_value``).  The
dense check is the oracle's ``dense_generalized_eigh`` (stands in for the
reference's ``dense_oracle``, eigensolver.py:396-425).

One SPEC claim does not hold for the reference itself, so it is pinned to the
reference's behaviour instead of to the SPEC text:

* path-5, k=2 "CV(proposed) < CV(le)": the reference's
  ``embed`` (embedding.py:77-103, K+1 pairs with the first dropped) gives
  CV 0.393 vs LE's 0.129.  The test asserts the GPU reproduces both CVs.

And one of the 50 random graphs (n=15, index 17 of the seed-2112 draw) makes
the reference's LOBPCG break down at seed 42 (Ritz sum to -1.7e13, 500
iterations, converged all False; checked against the reference package in
the build container).  For such runs the invariant tested is "converged
flags true => eigenpairs match the dense solve"; the monotone-Ritz-sum check
applies to converged runs.
"""

import numpy as np
import pytest

import oracle as O
from conftest import principal_angles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mg():
    import paper_2112_07862_b200 as mg
    return mg


def _random_family(count=50, seed=2112):
    """N in [10, 200], edge probability 3/N .. 10/N, connected."""
    from paper_2112_07862_b200 import synthetic
    rng = np.random.default_rng(seed)
    out = []
    for t in range(count):
        n = int(rng.integers(10, 201))
        p = rng.uniform(3.0, 10.0) / n
        extra = max(0, int(round(p * n * (n - 1) / 2)) - (n - 1))
        out.append(synthetic.random_connected(rng, n, extra, weighted=bool(t % 2)))
    return out


def _clusters(w, k, rel=1e-6):
    """Maximal runs of eigenvalues with gaps below rel*max|w| that end inside the
    first k (clusters cut by k are not comparable)."""
    scale = np.abs(w).max()
    out, i = [], 0
    while i < k:
        j = i + 1
        while j < w.size and w[j] - w[j - 1] < rel * scale:
            j += 1
        if j <= k:
            out.append((i, j))
        i = j
    return out


@pytest.fixture(scope="module")
def family_results(mg):
    res = []
    for g in _random_family():
        pair = mg.build_operator_pair(mg.Graph(*g))
        r = mg.lobpcg_smallest(pair.A, pair.B, mg.SolverConfig(k=4))
        a = O.CSR(pair.A.n, pair.A.indptr, pair.A.indices, pair.A.data)
        w, v = O.dense_generalized_eigh(a, pair.B.b, a.n)
        res.append((g, pair, r, w, v))
    return res


def test_oracle_equivalence_50_random_graphs(family_results):
    """SPEC.md:315 (acceptance 4): eigenvalues within 1e-8 relative
    of the dense solve, principal angles per cluster below 1e-6 rad."""
    n_conv = 0
    for g, pair, r, w, v in family_results:
        if not r.converged.all():
            continue
        n_conv += 1
        assert np.all(np.abs(r.eigenvalues - w[:4]) <= 1e-8 * np.abs(w[:4])), g[0]
        for i, j in _clusters(w, 4):
            ang = principal_angles(r.eigenvectors[:, i:j], v[:, i:j], pair.B.b).max()
            assert ang < 1e-6, (g[0], i, j, ang)
    assert n_conv >= 49


def test_nonconverged_matches_reference_breakdown(family_results):
    """The one graph the reference fails on (see module doc) is flagged
    non-converged here as well; nothing else is."""
    bad = [g[0] for g, _, r, _, _ in family_results if not r.converged.all()]
    assert bad in ([], [15])


def test_monotone_ritz_sum(family_results):
    """per iteration the block's Ritz sum is non-increasing (1e-12)."""
    for g, _, r, _, _ in family_results:
        if not r.converged.all():
            continue
        h = np.asarray(r.ritz_sum_history)
        assert h.size == r.iterations
        assert np.all(np.diff(h) <= 1e-12), (g[0], np.max(np.diff(h)))


def test_b_orthonormal_results(family_results):
    """every returned block is B-orthonormal."""
    for g, pair, r, _, _ in family_results:
        if not r.converged.all():
            continue
        x = r.eigenvectors
        gram = x.T @ (pair.B.b[:, None] * x)
        assert np.max(np.abs(gram - np.eye(x.shape[1]))) < 1e-10, g[0]


def test_trace_identity_full_block(mg):
    """with k = N the eigenvalue sum is trace(B^-1 A) (1e-9 rel)."""
    from paper_2112_07862_b200 import synthetic
    rng = np.random.default_rng(7)
    for n in (6, 9, 12):
        pair = mg.build_operator_pair(mg.Graph(*synthetic.random_connected(rng, n, n, weighted=True)))
        r = mg.lobpcg_smallest(pair.A, pair.B, mg.SolverConfig(k=n))
        tr = np.sum(pair.A.diagonal() / pair.B.b)
        assert abs(r.eigenvalues.sum() - tr) <= 1e-9 * abs(tr)


@pytest.mark.parametrize("kind,size,which,value", [("path", 2, "L", 2.0), ("ring", 4, "L", 2.0),
                                                   ("path", 5, "Q", 1.5)])
def test_fiedler_examples(mg, kind, size, which, value):
    """SPEC.md:310-312 (fiedler_value, eigensolver.py:463-468)."""
    from paper_2112_07862_b200 import synthetic
    g = mg.Graph(*synthetic.named(kind, size))
    m = mg.laplacian(g) if which == "L" else mg.two_hop_laplacian(mg.two_hop_sets(g))
    assert mg.fiedler_value(m) == pytest.approx(value, rel=1e-12)


def _cv(p, edges):
    d = np.array([np.linalg.norm(p[i] - p[j]) for i, j in edges])
    return d.std() / d.mean()


def test_embed_ring5_even_spacing(mg):
    """ring-5, k=2 -> consecutive-distance CV < 0.05."""
    from paper_2112_07862_b200 import synthetic
    e = mg.embed(mg.Graph(*synthetic.named("ring", 5)), 2)
    assert _cv(e.P, [(i, (i + 1) % 5) for i in range(5)]) < 0.05


def test_embed_path5_spacing_matches_reference(mg):
    """SPEC.md:365 claims CV(proposed) < CV(le) on path-5; the reference's own
    embed gives 0.3927 vs 0.1289 (module doc).  Pin the GPU to the oracle."""
    from paper_2112_07862_b200 import synthetic
    g = synthetic.named("path", 5)
    edges = [(i, i + 1) for i in range(4)]
    cv_p = _cv(mg.embed(mg.Graph(*g), 2).P, edges)
    cv_le = _cv(mg.laplacian_eigenmaps(mg.Graph(*g), 2).P, edges)
    assert cv_p == pytest.approx(_cv(O.embed(*g, 2)["P"], edges), rel=1e-8)
    assert cv_le == pytest.approx(_cv(O.laplacian_eigenmaps(*g, 2)["P"], edges), rel=1e-8)
    assert cv_p == pytest.approx(0.39273644209436437, rel=1e-6)
    assert cv_le == pytest.approx(0.12887141987909667, rel=1e-6)


def test_determinism_fp64_small(mg, family_results):
    """SPEC.md:318 / SURVEY §5: same input + seed -> bit-identical results."""
    for g, pair, r, _, _ in family_results[:10]:
        r2 = mg.lobpcg_smallest(pair.A, pair.B, mg.SolverConfig(k=4))
        assert r2.iterations == r.iterations
        assert np.array_equal(r2.eigenvalues, r.eigenvalues)
        assert np.array_equal(r2.eigenvectors, r.eigenvectors)
        assert r2.ritz_sum_history == r.ritz_sum_history


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_determinism_200k(mg, precision):
    """Bit-identical embeddings on the large path (CM reordering, tcgen05 Gram in
    fp32, staged Gram reductions): two runs of the C5 family at 200K points."""
    from paper_2112_07862_b200 import synthetic
    g = mg.Graph(*synthetic.config_graph("c5", n=200_000))
    cfg = mg.SolverConfig(k=17, tol=1e-4, max_iter=3000, seed=42, precision=precision)
    e1 = mg.embed(g, 16, cfg)
    e2 = mg.embed(g, 16, cfg)
    assert np.array_equal(e1.eigenvalues, e2.eigenvalues)
    assert np.array_equal(e1.P, e2.P)
