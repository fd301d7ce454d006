"""Graph.from_edges host logic (graph.py:31-79): canonical CSR and the
reference's validation messages.  Pure host code, no device needed."""

import numpy as np
import pytest

from paper_2112_07862_b200 import InputError
from paper_2112_07862_b200.core import Graph


def test_from_edges_canonical_csr():
    g = Graph.from_edges([(2, 0, 0.5), (0, 1), (3, 1, 2.0)])
    assert g.n == 4
    assert g.indptr.tolist() == [0, 2, 4, 5, 6]
    assert g.indices.tolist() == [1, 2, 0, 3, 0, 1]
    assert g.weights.tolist() == [1.0, 0.5, 1.0, 2.0, 0.5, 2.0]
    assert Graph.from_edges(np.array([[0, 1], [1, 2]])) == Graph.from_edges([(1, 2), (0, 1)])
    assert Graph.from_edges([], n=3).n == 3


@pytest.mark.parametrize("edges,n,msg", [
    ([(0, 1), (2, 2)], None, "self-loop on node 2"),
    ([(0, -1)], None, "negative node id in edge (0, -1)"),
    ([(0, 1, 0.0)], None, "edge (0, 1) has non-positive weight 0.0"),
    ([(0, 1, float("nan"))], None, "edge (0, 1) has non-positive weight nan"),
    ([(0, 1), (1, 0)], None, "duplicate edge {0, 1}"),
    ([(0, 5)], 3, "edge references node 5 >= n=3"),
])
def test_from_edges_errors(edges, n, msg):
    with pytest.raises(InputError) as e:
        Graph.from_edges(edges, n=n)
    assert str(e.value) == msg
