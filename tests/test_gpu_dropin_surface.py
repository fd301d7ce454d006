"""The rest of the drop-in type surface, on the device, against the reference.

SparseSymMatrix.frobenius_norm / row_sums / gershgorin / disc_left_ends /
from_scipy (sparse.py:35-98), Graph.degrees / adjacency / edge_array /
neighbor_weights / __eq__ (graph.py:88-137), balance_radii
(operators.py:189-202), and a reference-style caller (OperatorPair
.diagnostics as operators.py:76-85 writes it, via A.disc_left_ends()).
Goldens: tests/golden/scale_queries.* (make_golden_scale.py queries).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gold():
    z = np.load(os.path.join(GOLDEN, "scale_queries.npz"))
    with open(os.path.join(GOLDEN, "scale_queries.json")) as fh:
        return z, json.load(fh)


def _graph(mg, z, name):
    if f"{name}/graph_n" in z:
        return mg.Graph(int(z[f"{name}/graph_n"]), z[f"{name}/graph_ptr"], z[f"{name}/graph_idx"],
                        z[f"{name}/graph_w"])
    from paper_2112_07862_b200 import synthetic
    return mg.Graph(*synthetic.config_graph("c5", n=200_000))


@pytest.mark.parametrize("name", ["rand700", "grid", "c5_200K"])
def test_matrix_queries_bit_exact(gold, name):
    import paper_2112_07862_b200 as mg
    z, meta = gold
    g = _graph(mg, z, name)
    l = mg.laplacian(g)
    q = mg.two_hop_laplacian(mg.two_hop_sets(g))
    for key, m in (("L", l), ("Q", q)):
        rec = meta[name][key]
        assert m.frobenius_norm() == rec["frobenius_norm"]          # numpy pairwise sum, bit for bit
        rs = m.row_sums()
        c, r = m.gershgorin()
        left = m.disc_left_ends()
        assert sha(rs) == rec["sha_row_sums"]
        assert sha(c) == rec["sha_centers"] and sha(r) == rec["sha_radii"]
        assert sha(left) == rec["sha_left"]
        bs = mg.balance_radii(r)
        # log / exp differ from glibc's by an ulp at most; the means are numpy's sums
        assert abs(np.sum(bs.b) - rec["balance_b_sum"]) <= 1e-13 * rec["balance_b_sum"]
        assert bs.generalized_degree == pytest.approx(rec["balance_gdeg"], rel=1e-14)
        if f"{name}/{key}_balance_b" in z:
            ref = z[f"{name}/{key}_balance_b"]
            assert np.max(np.abs(bs.b - ref) / ref) < 4e-15
    assert sha(g.degrees()) == meta[name]["sha_degrees"]
    assert g.num_edges == meta[name]["num_edges"]


def test_graph_methods_and_reference_style_caller(gold):
    import scipy.sparse as sp
    import paper_2112_07862_b200 as mg
    z, _ = gold
    g = _graph(mg, z, "rand700")
    a = g.adjacency()
    assert isinstance(a, mg.SparseSymMatrix) and np.array_equal(a.data, g.weights)
    i, j, w = g.edge_array()
    assert np.all(i < j) and i.size == g.num_edges
    g2 = mg.Graph.from_edges(zip(i.tolist(), j.tolist(), w.tolist()), n=g.n)
    assert g2 == g and not (g2 == mg.Graph.from_edges([(0, 1)]))
    assert np.array_equal(g.neighbor_weights(5), g.weights[g.indptr[5]:g.indptr[6]])
    m = mg.SparseSymMatrix.from_scipy(sp.csr_matrix((a.data, a.indices, a.indptr), shape=(g.n, g.n)))
    assert np.array_equal(m.indptr, a.indptr) and np.array_equal(m.indices, a.indices)
    # operators.py:76-85 as the reference writes it, on the drop-in objects
    pair = mg.build_operator_pair(g)
    left = pair.A.disc_left_ends()
    binding = int(np.argmin(left))
    d = pair.diagnostics()
    assert d["binding_row"] == binding and d["min_disc_left_end"] == float(left[binding])
