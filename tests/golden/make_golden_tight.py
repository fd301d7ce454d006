"""Add tight (shift-invert) eigenpairs of the reference's C2 pair to c2.npz.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_tight.py

Uses the unmodified reference to build (A, B) and scipy eigsh (sigma=0) for
K+2 pairs (the extra one gives the gap above the block); stores the vectors
as float32 plus the reference's own per-column distance to them.
"""
import os
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")
import manigraph as mg  # noqa: E402

from paper_2112_07862_b200 import synthetic  # noqa: E402

g = synthetic.config_graph("c2")
pair = mg.build_operator_pair(mg.Graph(*g))
w, v = sla.eigsh(pair.A._csr, k=6, M=sp.diags(pair.B.b), sigma=0.0, which="LM", tol=1e-14)
o = np.argsort(w)
w, v = w[o], v[:, o]
for j in range(v.shape[1]):  # sign convention of eigensolver.py:83-89
    if v[np.argmax(np.abs(v[:, j])), j] < 0:
        v[:, j] = -v[:, j]
path = os.path.join(HERE, "c2.npz")
z = dict(np.load(path))
z["tight_eigenvalues6"] = w
z["tight_eigenvectors6"] = v.astype(np.float32)
np.savez_compressed(path, **z)
print("tight", w)
