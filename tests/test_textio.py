"""Text I/O: the native CSV / edge-list writers produce the
reference's bytes and the readers its values and errors (golden: the
unmodified reference's outputs, tests/golden/make_golden_io.py).  Host-only
code: these run in the CPU suite."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TMP = "/tmp/mgio_golden"  # the path the golden messages were recorded with


@pytest.fixture(scope="module")
def gio():
    with open(os.path.join(HERE, "golden", "io.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def mg():
    import paper_2112_07862_b200 as mg
    return mg


def test_save_embedding_csv_bytes(mg, gio, tmp_path):
    P = np.array(gio["P"], dtype=np.float64)
    P[0, 0] = -0.0  # JSON drops the sign of zero; the golden text has it
    path = tmp_path / "e.csv"
    for threads in (1, 3):
        mg.save_embedding_csv(P, path, threads=threads)
        assert path.read_text() == gio["emb_text"]


def test_load_embedding_csv_values(mg, gio, tmp_path):
    path = tmp_path / "e.csv"
    path.write_text(gio["emb_text"])
    Q = mg.load_embedding_csv(path)
    P = np.array(gio["P"])
    np.testing.assert_array_equal(Q, P)
    assert np.signbit(Q[0, 0])


def test_save_edge_list_bytes(mg, gio, tmp_path):
    gg = gio["graph"]
    g = mg.Graph(gg["n"], gg["indptr"], gg["indices"], gg["weights"])
    path = tmp_path / "edges.tsv"
    for threads in (1, 4):
        mg.save_edge_list(g, path, threads=threads)
        assert path.read_text() == gio["edge_text"]


def test_load_edge_list_arrays(mg, gio, tmp_path):
    path = tmp_path / "edges.tsv"
    path.write_text(gio["edge_text"])
    g = mg.load_edge_list(path)
    ref = gio["loaded"]
    assert g.n == ref["n"]
    np.testing.assert_array_equal(g.indptr, ref["indptr"])
    np.testing.assert_array_equal(g.indices, ref["indices"])
    np.testing.assert_array_equal(g.weights, ref["weights"])


@pytest.mark.parametrize("kind", ["edge", "emb"])
def test_malformed_inputs_match_reference_errors(mg, gio, kind):
    os.makedirs(TMP, exist_ok=True)
    for name, case in gio[f"{kind}_cases"].items():
        path = os.path.join(TMP, f"{kind}_{name}.{'txt' if kind == 'edge' else 'csv'}")
        with open(path, "w") as fh:
            fh.write(case["text"])
        load = mg.load_edge_list if kind == "edge" else mg.load_embedding_csv
        if case["ok"]:
            out = load(path)
            if kind == "edge":
                assert out.n == case["n"]
                np.testing.assert_array_equal(out.indptr, case["indptr"])
                np.testing.assert_array_equal(out.indices, case["indices"])
                np.testing.assert_array_equal(out.weights, case["weights"])
            else:
                np.testing.assert_array_equal(out, np.array(case["P"]))
            continue
        exc = getattr(mg, case["type"])
        with pytest.raises(exc) as ei:
            load(path)
        assert str(ei.value) == case["msg"], name
        if case["type"] == "ParseError":
            assert ei.value.lineno == case["lineno"] and ei.value.path == path


def test_large_round_trip(mg, tmp_path):
    """A 200K x 8 block through the multi-threaded writer and reader."""
    P = np.random.default_rng(2).normal(size=(200_000, 8)) * 1e3
    path = tmp_path / "big.csv"
    mg.save_embedding_csv(P, path)
    np.testing.assert_array_equal(mg.load_embedding_csv(path), P)
