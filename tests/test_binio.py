"""Binary embedding / graph files (csrc/mg_binio.cu): the
objects of the reference's text formats (embedding.py:131-166,
graph.py:147-194) round-trip bit for bit, multi-threaded, and corrupt or
non-canonical files fail like the reference's loaders (ParseError /
InputError).  Host-only code: these run in the CPU suite."""

import numpy as np
import pytest

import paper_2112_07862_b200 as mg
from paper_2112_07862_b200 import synthetic
from paper_2112_07862_b200.core import Embedding, Graph


@pytest.mark.parametrize("threads", [1, 5])
def test_embedding_roundtrip(tmp_path, threads):
    rng = np.random.default_rng(3)
    P = rng.standard_normal((70_001, 7))
    P[0, 0] = -0.0
    P[1, 1] = np.nan
    emb = Embedding(P=P, method="proposed", eigenvalues=rng.uniform(size=7),
                    b=rng.uniform(0.5, 2, size=70_001))
    path = tmp_path / "e.mgb"
    mg.save_embedding_bin(emb, path, threads=threads)
    back = mg.load_embedding_bin(path, threads=threads)
    assert back.method == "proposed"
    assert back.P.tobytes() == P.tobytes()
    assert np.array_equal(back.eigenvalues, emb.eigenvalues)
    assert np.array_equal(back.b, emb.b)
    # bare P (no eigenvalues / b)
    mg.save_embedding_bin(P[:10], path)
    back = mg.load_embedding_bin(path)
    assert back.b is None and back.P.tobytes() == P[:10].tobytes()
    assert np.all(np.isnan(back.eigenvalues))


def test_graph_roundtrip(tmp_path):
    g = Graph(*synthetic.config_graph("c5", n=30_000))
    path = tmp_path / "g.mgb"
    mg.save_graph_bin(g, path, threads=4)
    back = mg.load_graph_bin(path, threads=3)
    assert back == g


def test_bad_files(tmp_path):
    path = tmp_path / "x.mgb"
    path.write_bytes(b"not a file" * 10)
    with pytest.raises(mg.ParseError):
        mg.load_embedding_bin(path)
    with pytest.raises(mg.ParseError):
        mg.load_graph_bin(path)
    g = Graph.from_edges([(0, 1, 1.0), (1, 2, 2.0)])
    mg.save_graph_bin(g, path)
    mg.save_embedding_bin(np.zeros((3, 2)), tmp_path / "e.mgb")
    with pytest.raises(mg.ParseError):  # wrong kind
        mg.load_graph_bin(tmp_path / "e.mgb")
    # truncated
    data = path.read_bytes()
    (tmp_path / "t.mgb").write_bytes(data[:-8])
    with pytest.raises(mg.InputError, match="truncated"):
        mg.load_graph_bin(tmp_path / "t.mgb")
    # non-canonical: an asymmetric half-edge, a self-loop, a non-positive weight
    bad = Graph(3, g.indptr, g.indices, g.weights.copy())
    bad.weights[0] = 3.0
    mg.save_graph_bin(bad, path)
    with pytest.raises(mg.InputError, match="no matching"):
        mg.load_graph_bin(path)
    loop = Graph(2, np.array([0, 1, 1]), np.array([0]), np.array([1.0]))
    mg.save_graph_bin(loop, path)
    with pytest.raises(mg.InputError, match="self-loop on node 0"):
        mg.load_graph_bin(path)
    neg = Graph(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([-1.0, -1.0]))
    mg.save_graph_bin(neg, path)
    with pytest.raises(mg.InputError, match="non-positive weight"):
        mg.load_graph_bin(path)
