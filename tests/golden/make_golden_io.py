"""Golden text-I/O vectors from the UNMODIFIED reference (build container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Writes tests/golden/io.json: the reference's save_embedding_csv /
save_edge_list output text for seeded inputs, its load_edge_list arrays, and
for malformed inputs the exception class and message its loaders raise
(files under /tmp/mgio_golden/, the path the tests recreate).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from manigraph import embedding, graph  # noqa: E402  (the reference)

TMP = "/tmp/mgio_golden"

EDGE_CASES = {
    "ok_comments": "# header\n\n0 1 0.5\n1\t2\n  2 3 1e-3  \n# tail\n",
    "cols": "0 1\n1 2 3 4\n",
    "ints": "0 1\nx 2\n",
    "weight": "0 1 abc\n",
    "selfloop": "0 1\n2 2 1.0\n",
    "negative": "0 1\n-1 2\n",
    "nonpos": "0 1 0\n",
    "negw": "0 1\n1 2 -2.5\n",
    "dup": "0 1\n2 3\n1 0 2.0\n",
    "empty": "# nothing\n\n",
}
EMB_CASES = {
    "header": "id,c1\n0,1.0\n",
    "ragged": "node,c1,c2\n0,1,2\n1,3\n",
    "dense": "node,c1\n0,1.5\n2,2.5\n",
    "float": "node,c1\n0,1.5\n1,abc\n",
    "shuffled": "node,c1,c2\n2,5,6\n0,1,2\n1,3,4\n",
}


def main():
    os.makedirs(TMP, exist_ok=True)
    g = np.random.default_rng(4)
    P = g.normal(size=(9, 4)) * np.logspace(-8, 8, 4)
    P[0, 0] = -0.0
    P[1, 1] = 5e-324
    P[2, 2] = 1e300
    P[3, 3] = 0.1
    emb_path = os.path.join(TMP, "emb.csv")
    embedding.save_embedding_csv(embedding.Embedding(P=P, method="x", eigenvalues=np.zeros(4)),
                                 emb_path)
    n = 12
    edges = [(i, j, float(w)) for i, j, w in
             zip(g.integers(0, n, 40), g.integers(0, n, 40), g.uniform(0.01, 3, 40))]
    seen, uniq = set(), []
    for i, j, w in edges:
        if i != j and (min(i, j), max(i, j)) not in seen:
            seen.add((min(i, j), max(i, j)))
            uniq.append((int(i), int(j), w))
    G = graph.Graph.from_edges(uniq, n=n)
    edge_path = os.path.join(TMP, "edges.tsv")
    graph.save_edge_list(G, edge_path)
    G2 = graph.load_edge_list(edge_path)
    out = {
        "P": P.tolist(), "emb_text": open(emb_path).read(),
        "graph": {"n": G.n, "indptr": G.indptr.tolist(), "indices": G.indices.tolist(),
                  "weights": G.weights.tolist()},
        "edge_text": open(edge_path).read(),
        "loaded": {"n": G2.n, "indptr": G2.indptr.tolist(), "indices": G2.indices.tolist(),
                   "weights": G2.weights.tolist()},
        "edge_cases": {}, "emb_cases": {},
    }
    for name, text in EDGE_CASES.items():
        path = os.path.join(TMP, f"edge_{name}.txt")
        open(path, "w").write(text)
        try:
            gg = graph.load_edge_list(path)
            out["edge_cases"][name] = {"text": text, "ok": True, "n": gg.n,
                                       "indptr": gg.indptr.tolist(),
                                       "indices": gg.indices.tolist(),
                                       "weights": gg.weights.tolist()}
        except Exception as e:  # noqa: BLE001
            out["edge_cases"][name] = {"text": text, "ok": False, "type": type(e).__name__,
                                       "msg": str(e), "lineno": getattr(e, "lineno", None)}
    for name, text in EMB_CASES.items():
        path = os.path.join(TMP, f"emb_{name}.csv")
        open(path, "w").write(text)
        try:
            Q = embedding.load_embedding_csv(path)
            out["emb_cases"][name] = {"text": text, "ok": True, "P": Q.tolist()}
        except Exception as e:  # noqa: BLE001
            out["emb_cases"][name] = {"text": text, "ok": False, "type": type(e).__name__,
                                      "msg": str(e)}
    json.dump(out, open(os.path.join(HERE, "io.json"), "w"), indent=0)
    print("wrote io.json")


if __name__ == "__main__":
    main()
