"""Golden k-means / normalize_rows / RNG vectors from the UNMODIFIED reference
(build container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_kmeans.py

Writes tests/golden/kmeans.npz: inputs (seeded numpy blobs, an embedding-like
block, duplicate points that force the empty-cluster repair) and the
reference's labels (manigraph.clustering.kmeans), normalize_rows outputs and
the first draws of its xoshiro256** streams (manigraph.rng).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from manigraph import clustering, rng  # noqa: E402  (the reference)


def main():
    out = {}
    g = np.random.default_rng(7)
    cases = []
    # well separated blobs
    centers = g.uniform(-10, 10, size=(5, 3))
    x = np.concatenate([c + g.normal(0, 0.5, size=(200, 3)) for c in centers])
    cases.append(("blobs", x, 5, 5, 42))
    # overlapping blobs (ties and restarts matter)
    x = np.concatenate([c + g.normal(0, 3.0, size=(150, 2)) for c in g.uniform(-5, 5, (4, 2))])
    cases.append(("overlap", x, 4, 8, 3))
    # embedding-like rows: 10 indicator-ish clusters in 17 dims
    lab = g.integers(0, 10, 3000)
    basis = g.normal(size=(10, 17))
    x = basis[lab] + g.normal(0, 0.05, size=(3000, 17))
    cases.append(("embed17", x, 10, 20, 42))
    # many duplicate points: forces the empty-cluster repair
    x = np.concatenate([np.zeros((50, 2)), np.ones((3, 2)), g.normal(size=(5, 2))])
    cases.append(("dups", x, 6, 4, 11))
    names = []
    for name, x, c, r, seed in cases:
        names.append(name)
        out[f"{name}_x"] = x
        out[f"{name}_meta"] = np.array([c, r, seed])
        out[f"{name}_labels"] = clustering.kmeans(x, c, restarts=r, seed=seed, threads=1)
        out[f"{name}_norm"] = clustering.normalize_rows(x)
    out["names"] = np.array(names)
    # RNG streams
    draws = []
    for seed, idx in [(42, 0), (42, 19), (0, 0), (2**63 + 5, 3)]:
        gen = rng.Xoshiro256(rng.stream_seed(seed, idx))
        draws.append([gen.next_u64() for _ in range(8)])
    out["rng_draws"] = np.array(draws, dtype=np.uint64)
    out["rng_seeds"] = np.array([[42, 0], [42, 19], [0, 0], [2**63 + 5, 3]], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), **out)
    print("wrote kmeans.npz:", names)


if __name__ == "__main__":
    main()
