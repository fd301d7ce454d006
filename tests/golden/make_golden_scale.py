"""Reference-generated goldens at the benchmarked scales (C3, C4, C5 families).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scale.py NAME [NAME ...]

NAME is one of ``c3_1M c3_100K c4_500K c5_1M c5_2M c5_200K hub defl2 queries``.  Runs the
UNMODIFIED reference (``manigraph`` from /root/reference/pkg/src, build
container only) on the harness graphs of ``paper_2112_07862_b200.synthetic``
and writes ``scale_<NAME>.json`` (+ ``scale_<NAME>.npz`` for small arrays):

* graph hashes (so the GPU box can check it rebuilt the same graph);
* sha256 of the T / Q / A indptr, indices and values exactly as the reference
  computed them (operators.py:88-135, 179-186; A assembled with the
  reference's own eps and mu), eps (operators.py:138-156, the 60-iteration
  best-effort LOBPCG of eigensolver.py:431-460), mu, diagnostics, and b
  (operators.py:189-219) at 8192 fixed sampled rows plus its sum / sum of
  squares / dot with a fixed random vector (b is reproduced to ~1e-15, not
  bit for bit, so a hash would not do);
* for ``c5_200K`` and ``c3_100K``: tight generalized eigenpairs of the reference's (A, B)
  (scipy eigsh shift-invert, tol 1e-12; vectors stored as float32, the
  sign convention of eigensolver.py:83-89) and the reference's own
  ``lobpcg_smallest`` at the config tolerance (eigenvalues, iterations, and
  its per-cluster distance to the tight vectors);
* for ``c4_500K``: the reference's embedding readout (``lobpcg_smallest`` on
  the pair, bypassing _check_embeddable as SURVEY 8(c).6 prescribes, then the
  reference's ``normalize_rows`` + ``kmeans`` with 10 clusters on the first
  10 columns) -> labels, stored as the label of each patch's points;
* ``hub``: a 700-leaf star plus a sparse random graph among the leaves, so
  every leaf row of adj*adj has more than 512 products and the GPU two-hop
  builder takes its large-row tier (mg_graph.cu); full arrays stored.

/root/reference does not exist on the GPU box: these files are what the
``-m gpu`` tests read there.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import manigraph as mg  # noqa: E402  (the reference)

from paper_2112_07862_b200 import synthetic  # noqa: E402

CASES = {
    # name: (config, n, solve)
    "c3_1M": ("c3", 1_000_000, False),
    "c4_500K": ("c4", 500_000, False),
    "c5_1M": ("c5", 1_000_000, False),
    "c5_2M": ("c5", 2_000_000, False),
    "c5_200K": ("c5", 200_000, True),
    "c3_100K": ("c3", 100_000, True),
}
B_SAMPLE = 8192


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def b_summary(b):
    n = b.size
    rows = np.unique(np.random.default_rng(1234).integers(0, n, size=B_SAMPLE))
    v = np.random.default_rng(4321).standard_normal(n)
    return rows, {"sum": float(np.sum(b)), "sumsq": float(np.sum(b * b)),
                  "dot_rand4321": float(v @ b), "min": float(b.min()), "max": float(b.max())}


def graph_meta(g):
    n, ptr, idx, w = g
    return {"n": int(n), "nnz": int(idx.size), "sha_indptr": sha(ptr), "sha_indices": sha(idx),
            "sha_weights": sha(w)}


def pair_meta(G, out, meta):
    tt = {}
    t0 = time.perf_counter()
    l = mg.laplacian(G)
    tt["laplacian"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    t = mg.two_hop_sets(G)
    tt["two_hop_sets"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    q = mg.two_hop_laplacian(t)
    tt["two_hop_laplacian"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    eps = mg.identity_shift(q, solver_seed=42)
    tt["identity_shift"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    mu = mg.repulsion_weight(l, q, eps)
    a = mg.assemble_operator(l, q, mu, eps)
    tt["mu_assemble"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    bs = mg.degree_balancing(a)
    tt["degree_balancing"] = time.perf_counter() - t0
    pair = mg.OperatorPair(A=a, B=bs, mu=mu, epsilon=eps, Q=q)
    rows, bstat = b_summary(bs.b)
    out["b_rows"] = rows
    out["b_at_rows"] = bs.b[rows]
    meta["pair"] = {
        "eps": float(eps), "mu": float(mu), "diagnostics": pair.diagnostics(),
        "generalized_degree": float(bs.generalized_degree), "b_stats": bstat,
        "T_nnz": int(t.indices.size), "Q_nnz": int(q.nnz), "A_nnz": int(a.nnz),
        "L_nnz": int(l.nnz),
        "sha_L_ptr": sha(l.indptr), "sha_L_idx": sha(l.indices), "sha_L_val": sha(l.data),
        "sha_T_ptr": sha(t.indptr), "sha_T_idx": sha(t.indices),
        "sha_Q_ptr": sha(q.indptr), "sha_Q_idx": sha(q.indices), "sha_Q_val": sha(q.data),
        "sha_A_ptr": sha(a.indptr), "sha_A_idx": sha(a.indices), "sha_A_val": sha(a.data),
        "seconds": tt,
        # reference dtypes, so the GPU side hashes the same bytes
        "dtypes": {"ptr": str(a.indptr.dtype), "idx": str(a.indices.dtype), "val": str(a.data.dtype)},
    }
    return pair


def fix_signs(v):
    for j in range(v.shape[1]):  # eigensolver.py:83-89
        if v[np.argmax(np.abs(v[:, j])), j] < 0:
            v[:, j] = -v[:, j]
    return v


def principal_angles_b(U, V, b):
    s = np.sqrt(b)[:, None]
    qu, _ = np.linalg.qr(U * s)
    qv, _ = np.linalg.qr(V * s)
    m = qv - qu @ (qu.T @ qv)
    ss = np.linalg.svd(m, compute_uv=False)
    return np.arcsin(np.clip(np.sort(ss)[::-1], 0.0, 1.0))


def tight_and_solve(name, c, pair, out, meta):
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    k = c.k + 1
    t0 = time.perf_counter()
    w, v = sla.eigsh(pair.A._csr, k=k + 1, M=sp.diags(pair.B.b), sigma=0.0, which="LM", tol=1e-12)
    o = np.argsort(w)
    w, v = w[o], fix_signs(v[:, o])
    meta["tight"] = {"method": "scipy.sparse.linalg.eigsh shift-invert sigma=0 tol=1e-12, k=K+2",
                     "seconds": time.perf_counter() - t0, "eigenvalues": w.tolist()}
    out["tight_eigenvalues"] = w
    out["tight_eigenvectors"] = v[:, :k].astype(np.float32)
    cfg = mg.SolverConfig(k=k, tol=c.tol, max_iter=c.max_iter, seed=42)
    t0 = time.perf_counter()
    res = mg.lobpcg_smallest(pair.A, pair.B, cfg)
    b = pair.B.b
    ang = [float(principal_angles_b(res.eigenvectors[:, [j]], v[:, [j]], b)[0]) for j in range(k)]
    # clusters of the tight spectrum (relative gap < 1e-2); a cluster is
    # complete when it ends before the block edge (gap to eigenvalue k+1)
    cl, cur = [], [0]
    for i in range(1, k + 1):
        if w[i] - w[i - 1] < 1e-2 * abs(w[i]):
            cur.append(i)
        else:
            cl.append(cur)
            cur = [i]
    cl.append(cur)
    complete = [c_ for c_ in cl if c_[-1] < k]
    cang = [float(principal_angles_b(res.eigenvectors[:, c_], v[:, c_], b).max()) for c_ in complete]
    meta["clusters"] = {"rule": "tight eigenvalues, relative gap < 1e-2; complete = ends below column k",
                        "complete": complete, "ref_angle_per_cluster": cang}
    meta["solve"] = {"iterations": int(res.iterations), "k": k, "tol": c.tol,
                     "max_iter": c.max_iter, "seconds": time.perf_counter() - t0,
                     "eigenvalues": res.eigenvalues.tolist(),
                     "converged": [bool(x) for x in res.converged],
                     "angle_to_tight_per_column": ang}
    out["ref_eigenvalues"] = res.eigenvalues
    return res


def c4_labels(c, pair, n, out, meta):
    from manigraph import clustering
    k = c.k + 1
    cfg = mg.SolverConfig(k=k, tol=c.tol, max_iter=c.max_iter, seed=42)
    t0 = time.perf_counter()
    res = mg.lobpcg_smallest(pair.A, pair.B, cfg)
    x = clustering.normalize_rows(res.eigenvectors[:, :10])
    labels = np.asarray(clustering.kmeans(x, 10))  # clustering.py:101-106 defaults
    per = n // 10
    out["ref_labels_first_per_patch"] = labels[::per][:10]
    truth = np.arange(n) // per
    same = len(set(zip(labels.tolist(), truth.tolist()))) == 10 == len(set(labels.tolist()))
    meta["solve"] = {"iterations": int(res.iterations), "k": k, "tol": c.tol,
                     "seconds": time.perf_counter() - t0, "eigenvalues": res.eigenvalues.tolist(),
                     "converged": [bool(x) for x in res.converged],
                     "labels_equal_patches_up_to_permutation": bool(same),
                     "labels_sha": sha(np.asarray(labels, np.int64))}


def make_case(name):
    cname, n, solve = CASES[name]
    c = synthetic.CONFIGS[cname]
    out, meta = {}, {"config": cname, "n": n, "reference": "manigraph (unmodified, /root/reference/pkg/src)"}
    t0 = time.perf_counter()
    g = synthetic.config_graph(cname, n=n)
    meta["graph"] = graph_meta(g)
    meta["graph"]["seconds"] = time.perf_counter() - t0
    G = mg.Graph(*g)
    pair = pair_meta(G, out, meta)
    save(name, out, meta)  # structure goldens first: the solves below are long
    print(name, "pair", json.dumps(meta["pair"]["seconds"]), flush=True)
    if solve:
        tight_and_solve(name, c, pair, out, meta)
        save(name, out, meta)
    if cname == "c4":
        c4_labels(c, pair, n, out, meta)
        save(name, out, meta)
    print(name, "done", flush=True)


def make_hub():
    """Star with 700 leaves + a random sparse graph among the leaves (weighted)."""
    rng = np.random.default_rng(777)
    n = 701
    lo = [0] * 700
    hi = list(range(1, 701))
    keys = set()
    while len(keys) < 1400:
        i, j = sorted(int(x) for x in rng.integers(1, n, size=2))
        if i != j:
            keys.add((i, j))
    for i, j in sorted(keys):
        lo.append(i)
        hi.append(j)
    w = rng.uniform(0.5, 2.0, size=len(lo))
    g = synthetic.from_edges(n, lo, hi, w)
    G = mg.Graph(*g)
    out, meta = {}, {"reference": "manigraph (unmodified)"}
    out["graph_ptr"], out["graph_idx"], out["graph_w"] = g[1], g[2], g[3]
    out["graph_n"] = np.int64(n)
    l = mg.laplacian(G)
    t = mg.two_hop_sets(G)
    q = mg.two_hop_laplacian(t)
    ql = mg.two_hop_laplacian(t, literal_diagonal=True)
    eps = mg.identity_shift(q, solver_seed=42)
    mu = mg.repulsion_weight(l, q, eps)
    a = mg.assemble_operator(l, q, mu, eps)
    bs = mg.degree_balancing(a)
    for key, m in (("T", t), ("Q", q), ("QL", ql), ("A", a)):
        out[f"{key}_ptr"], out[f"{key}_idx"] = m.indptr, m.indices
        if key != "T":
            out[f"{key}_val"] = m.data
    out["b"] = bs.b
    deg = np.diff(g[1])
    prod = np.array([deg[g[2][g[1][i]:g[1][i + 1]]].sum() for i in range(n)])
    meta.update(eps=float(eps), mu=float(mu), max_products_per_row=int(prod.max()),
                rows_over_512_products=int((prod > 512).sum()))
    save("hub", out, meta)
    print("hub", meta, flush=True)


def make_defl():
    """lobpcg_smallest with a two-column deflation block (eigensolver.py:179-184,
    239-241): the graph Laplacian of a random weighted graph, B = b of its pair,
    deflating its two lowest generalized eigenvectors (so the deflated solve converges
    to pairs 3..6, also checked against dense eigh)."""
    g = synthetic.random_connected(np.random.default_rng(31), 300, extra=600, weighted=True)
    G = mg.Graph(*g)
    l = mg.laplacian(G)
    n = g[0]
    b = np.random.default_rng(32).uniform(0.5, 2.0, size=n)
    import scipy.linalg as sl
    dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(l.indptr))
    dense[rows, l.indices] = l.data
    wd, vd = sl.eigh(dense, np.diag(b))
    # the two lowest generalized eigenvectors (the constant null vector and the
    # Fiedler vector), unnormalised so the projections carry y'By denominators
    y = np.stack([np.full(n, 1 / np.sqrt(n)), 3.0 * vd[:, 1]], axis=1)
    out_dense = wd[:8]
    cfg = mg.SolverConfig(k=4, tol=1e-9, max_iter=1000, seed=42)
    res = mg.lobpcg_smallest(l, b, cfg, deflate=y)
    out = {"graph_ptr": g[1], "graph_idx": g[2], "graph_w": g[3], "graph_n": np.int64(n), "b": b,
           "deflate": y, "eigenvalues": res.eigenvalues, "eigenvectors": res.eigenvectors,
           "converged": res.converged, "dense_eigenvalues": out_dense}
    meta = {"reference": "manigraph (unmodified)", "iterations": int(res.iterations),
            "k": 4, "tol": 1e-9, "max_iter": 1000, "seed": 42}
    save("defl2", out, meta)
    print("defl2", meta, res.eigenvalues, flush=True)


def make_queries():
    """SparseSymMatrix.frobenius_norm / row_sums / gershgorin / disc_left_ends,
    Graph.degrees / edge_array, balance_radii (sparse.py:76-98, graph.py:93-102,
    operators.py:189-202) on the reference's own matrices: small graphs in full,
    the C5-family 200K operator as hashes (its frobenius norm exercises numpy's
    pairwise-summation tree far past one 128-element block)."""
    out, meta = {}, {"reference": "manigraph (unmodified)"}
    cases = {"rand700": synthetic.random_connected(np.random.default_rng(99), 700, extra=900,
                                                   weighted=True),
             "grid": synthetic.named("grid", (30, 40)),
             "c5_200K": synthetic.config_graph("c5", n=200_000)}
    for name, g in cases.items():
        G = mg.Graph(*g)
        l = mg.laplacian(G)
        q = mg.two_hop_laplacian(mg.two_hop_sets(G))
        rec = {}
        for key, m in (("L", l), ("Q", q)):
            c, r = m.gershgorin()
            rec[key] = {"frobenius_norm": m.frobenius_norm(), "sha_row_sums": sha(m.row_sums()),
                        "sha_centers": sha(c), "sha_radii": sha(r),
                        "sha_left": sha(m.disc_left_ends()), "trace": m.trace()}
            bs = mg.operators.balance_radii(r)
            rec[key]["balance_b_sum"] = float(np.sum(bs.b))
            rec[key]["balance_gdeg"] = float(bs.generalized_degree)
            if g[0] <= 5000:
                out[f"{name}/{key}_row_sums"] = m.row_sums()
                out[f"{name}/{key}_radii"] = r
                out[f"{name}/{key}_left"] = m.disc_left_ends()
                out[f"{name}/{key}_balance_b"] = bs.b
        rec["sha_degrees"] = sha(G.degrees())
        rec["num_edges"] = G.num_edges
        if g[0] <= 5000:
            out[f"{name}/degrees"] = G.degrees()
            out[f"{name}/graph_ptr"], out[f"{name}/graph_idx"], out[f"{name}/graph_w"] = g[1], g[2], g[3]
            out[f"{name}/graph_n"] = np.int64(g[0])
        meta[name] = rec
    save("queries", out, meta)
    print("queries", json.dumps(meta)[:400], flush=True)


def save(name, out, meta):
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), **out)
    with open(os.path.join(HERE, f"scale_{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    for what in sys.argv[1:]:
        if what == "hub":
            make_hub()
        elif what == "defl2":
            make_defl()
        elif what == "queries":
            make_queries()
        else:
            make_case(what)
