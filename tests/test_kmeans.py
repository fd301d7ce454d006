"""k-means / normalize_rows (the C4 readout): the oracle
restatement is pinned to the reference's outputs (tests/golden/kmeans.npz from
tests/golden/make_golden_kmeans.py), then the device path is compared with it.
"""

import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gk():
    return np.load(os.path.join(HERE, "golden", "kmeans.npz"))


def test_oracle_rng_streams_match_reference(gk):
    for (seed, idx), draws in zip(gk["rng_seeds"].tolist(), gk["rng_draws"].tolist()):
        g = O.Xoshiro256(O.stream_seed(int(seed), int(idx)))
        assert [g.next_u64() for _ in range(8)] == [int(v) for v in draws]


def test_oracle_kmeans_matches_reference(gk):
    for name in gk["names"].tolist():
        c, r, seed = (int(v) for v in gk[f"{name}_meta"])
        lab, _ = O.kmeans(gk[f"{name}_x"], c, restarts=r, seed=seed)
        np.testing.assert_array_equal(lab, gk[f"{name}_labels"], err_msg=name)
        np.testing.assert_array_equal(O.normalize_rows(gk[f"{name}_x"]), gk[f"{name}_norm"])


@pytest.mark.gpu
def test_device_kmeans_matches_reference(gk):
    import paper_2112_07862_b200 as mg
    for name in gk["names"].tolist():
        c, r, seed = (int(v) for v in gk[f"{name}_meta"])
        lab = mg.kmeans(gk[f"{name}_x"], c, restarts=r, seed=seed)
        # identical labels (same seeding draws, same Lloyd fixed point); ties at
        # the 1e-16 level are the only way these could differ (mg_kmeans.cu)
        np.testing.assert_array_equal(lab, gk[f"{name}_labels"], err_msg=name)
        np.testing.assert_allclose(mg.normalize_rows(gk[f"{name}_x"]), gk[f"{name}_norm"],
                                   rtol=1e-15, atol=1e-300)


@pytest.mark.gpu
def test_device_kmeans_errors_and_trivial_cases():
    import paper_2112_07862_b200 as mg
    x = np.random.default_rng(0).normal(size=(20, 3))
    with pytest.raises(mg.InputError):
        mg.kmeans(x, 0)
    with pytest.raises(mg.InputError):
        mg.kmeans(x, 21)
    with pytest.raises(mg.InputError):
        mg.kmeans(x, 3, restarts=0)
    np.testing.assert_array_equal(mg.kmeans(x, 1), np.zeros(20, np.int64))
    np.testing.assert_array_equal(mg.kmeans(x, 20), np.arange(20))


@pytest.mark.gpu
def test_device_kmeans_large_vs_oracle():
    """200K rows x 17 (C4-like embedding rows): same partition as the oracle."""
    import paper_2112_07862_b200 as mg
    g = np.random.default_rng(5)
    lab = g.integers(0, 10, 200_000)
    x = g.normal(size=(10, 17))[lab] + g.normal(0, 0.2, size=(200_000, 17))
    dev = mg.kmeans(x, 10, restarts=3, seed=42)
    ref, _ = O.kmeans(x, 10, restarts=3, seed=42)
    np.testing.assert_array_equal(dev, ref)
