"""Golden kNN graphs from the UNMODIFIED reference's knn_graph (graph.py:281-315),
build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_knn.py

Writes tests/golden/knn.npz: the inputs and the reference Graph arrays.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import manigraph as ref  # noqa: E402  (the reference)

from paper_2112_07862_b200 import synthetic  # noqa: E402


def main():
    g = np.random.default_rng(3)
    lattice = np.stack(np.meshgrid(np.arange(15.0), np.arange(12.0)), -1).reshape(-1, 2)
    cases = [
        ("c1", synthetic.points("c1"), 10, True),             # config 1 point cloud
        ("cube3d", g.uniform(size=(700, 3)), 8, True),
        ("lattice", lattice, 4, True),                         # exact distance ties
        ("lattice_unw", lattice, 6, False),
        ("swiss", synthetic.points("c2", n=1500), 10, True),
        ("dim17", g.normal(size=(400, 17)), 7, True),
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
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "knn.npz"), **out)
    print("wrote knn.npz:", names)


if __name__ == "__main__":
    main()
