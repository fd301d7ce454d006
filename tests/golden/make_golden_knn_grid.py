"""Golden kNN graphs above the device grid search's threshold (n >= 4096, d <= 3)
from the UNMODIFIED reference's knn_graph (graph.py:281-315), build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_knn_grid.py

Cases: a uniform 3-D cloud, a 2-D lattice (exact distance ties: lower index
wins), 1-D points, and two far-apart Gaussian blobs (empty cells, long
searches).  Writes tests/golden/knn_grid.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import manigraph as ref  # noqa: E402  (the reference)


def main():
    g = np.random.default_rng(17)
    lattice = np.stack(np.meshgrid(np.arange(80.0), np.arange(70.0)), -1).reshape(-1, 2)
    blobs = np.concatenate([g.normal(size=(3000, 3)) * 0.05, g.normal(size=(3000, 3)) * 0.2 + 4.0])
    cases = [
        ("cube20k", g.uniform(size=(20000, 3)), 8, True),
        ("lattice5600", lattice, 4, True),
        ("line6000", np.sort(g.uniform(size=(6000, 1)), axis=0)[::-1].copy(), 6, True),
        ("blobs6000", blobs, 10, True),
    ]
    out, names = {}, []
    for name, x, k, wt in cases:
        gr = ref.knn_graph(x, k, weighted=wt)
        names.append(name)
        out[f"{name}_x"] = x
        out[f"{name}_k"] = np.array([k, int(wt)])
        out[f"{name}_indptr"] = gr.indptr
        out[f"{name}_indices"] = gr.indices
        out[f"{name}_weights"] = gr.weights
        print(name, gr.n, gr.indices.size, flush=True)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "knn_grid.npz"), **out)


if __name__ == "__main__":
    main()
