"""Generate golden vectors by running the UNMODIFIED reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [small|c1|c2|all]

Imports ``manigraph`` from /root/reference/pkg/src (read-only; never shipped)
and records its outputs on seeded inputs produced by this repo's harness
(``paper_2112_07862_b200.synthetic``).  The fixtures written next to this
script (``*.npz``) are what ``tests/test_oracle_golden.py`` pins the oracle
against and what the GPU parity tests compare with; /root/reference does not
exist on the GPU box, so nothing at test time reads it.
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
from manigraph import eigensolver as ref_es  # noqa: E402

from paper_2112_07862_b200 import synthetic  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_graph(g):
    n, ptr, idx, w = g
    return mg.Graph(n, ptr, idx, w)


def pair_record(prefix, g, out, meta, seed=42):
    G = ref_graph(g)
    l = mg.laplacian(G)
    t = mg.two_hop_sets(G)
    q = mg.two_hop_laplacian(t)
    ql = mg.two_hop_laplacian(t, literal_diagonal=True)
    rec = {}
    out[f"{prefix}/L_ptr"], out[f"{prefix}/L_idx"], out[f"{prefix}/L_val"] = l.indptr, l.indices, l.data
    out[f"{prefix}/T_ptr"], out[f"{prefix}/T_idx"] = t.indptr, t.indices
    out[f"{prefix}/Q_ptr"], out[f"{prefix}/Q_idx"], out[f"{prefix}/Q_val"] = q.indptr, q.indices, q.data
    out[f"{prefix}/QL_ptr"], out[f"{prefix}/QL_idx"], out[f"{prefix}/QL_val"] = ql.indptr, ql.indices, ql.data
    try:
        eps = mg.identity_shift(q, solver_seed=seed)
        mu = mg.repulsion_weight(l, q, eps)
        a = mg.assemble_operator(l, q, mu, eps)
        out[f"{prefix}/A_ptr"], out[f"{prefix}/A_idx"], out[f"{prefix}/A_val"] = a.indptr, a.indices, a.data
        rec.update(eps=float(eps), mu=float(mu))
        try:
            bs = mg.degree_balancing(a)
            out[f"{prefix}/b"] = bs.b
            rec["generalized_degree"] = float(bs.generalized_degree)
            pair = mg.OperatorPair(A=a, B=bs, mu=mu, epsilon=eps, Q=q)
            rec["diagnostics"] = pair.diagnostics()
        except mg.DisconnectedGraphError as e:
            rec["b_error"] = "DisconnectedGraphError: " + str(e)
    except mg.InputError as e:
        rec["pair_error"] = "InputError: " + str(e)
    meta[prefix] = rec
    return rec


def embed_record(prefix, g, k, cfg, out, meta, le=False):
    G = ref_graph(g)
    t0 = time.perf_counter()
    fn = mg.laplacian_eigenmaps if le else mg.embed
    try:
        emb = fn(G, k, cfg, require_convergence=False)
    except mg.ManigraphError as e:
        meta[prefix] = {"error": type(e).__name__, "message": str(e),
                        "n_components": getattr(e, "n_components", None)}
        return
    dt = time.perf_counter() - t0
    out[f"{prefix}/P"] = emb.P
    out[f"{prefix}/eigenvalues"] = emb.eigenvalues
    d = dict(emb.diagnostics)
    meta[prefix] = {"diagnostics": d, "seconds": dt, "k": k,
                    "tol": cfg.tol, "max_iter": cfg.max_iter, "seed": cfg.seed}


def lobpcg_record(prefix, a, b, cfg, out, meta, deflate=None):
    res = mg.lobpcg_smallest(a, b, cfg, deflate=deflate)
    out[f"{prefix}/eigenvalues"] = res.eigenvalues
    out[f"{prefix}/eigenvectors"] = res.eigenvectors
    out[f"{prefix}/residual_norms"] = res.residual_norms
    out[f"{prefix}/converged"] = res.converged
    out[f"{prefix}/history"] = np.asarray(res.ritz_sum_history)
    meta[prefix] = {"iterations": int(res.iterations), "k": cfg.k, "tol": cfg.tol,
                    "max_iter": cfg.max_iter, "seed": cfg.seed}


def make_small():
    out, meta = {}, {}
    named = {
        "path5": synthetic.named("path", 5), "path10": synthetic.named("path", 10),
        "star4": synthetic.named("star", 4), "complete5": synthetic.named("complete", 5),
        "ring6": synthetic.named("ring", 6), "ring9": synthetic.named("ring", 9),
        "grid4x5": synthetic.named("grid", (4, 5)),
    }
    rng = np.random.default_rng(20251020)
    for i in range(12):
        n = int(rng.integers(5, 200))
        named[f"rand{i}"] = synthetic.random_connected(rng, n, weighted=bool(i % 2))
    # isolated node (DisconnectedGraphError from degree balancing, operators.py:212)
    named["isolated3"] = synthetic.from_edges(3, [0], [1], [1.0])
    # two components (embed raises DisconnectedGraphError with n_components)
    named["twocomp"] = synthetic.from_edges(6, [0, 1, 3, 4], [1, 2, 4, 5], [1.0, 2.0, 1.0, 0.5])
    for name, g in named.items():
        out[f"{name}/graph_ptr"], out[f"{name}/graph_idx"], out[f"{name}/graph_w"] = g[1], g[2], g[3]
        out[f"{name}/graph_n"] = np.int64(g[0])
        pair_record(f"{name}/pair", g, out, meta)
    embed_cases = [("path5", 1), ("path5", 2), ("ring6", 2), ("ring9", 3), ("grid4x5", 3),
                   ("path10", 2), ("star4", 1), ("twocomp", 1)]
    embed_cases += [(f"rand{i}", 2 + i % 3) for i in range(12)]
    for name, k in embed_cases:
        cfg = mg.SolverConfig(k=k + 1, tol=1e-8, max_iter=500, seed=42)
        embed_record(f"{name}/embed{k}", named[name], k, cfg, out, meta)
    for name, k in [("path10", 2), ("ring9", 2), ("rand3", 3)]:
        cfg = mg.SolverConfig(k=k + 1, tol=1e-8, max_iter=500, seed=7)
        embed_record(f"{name}/le{k}", named[name], k, cfg, out, meta, le=True)
    # SPEC.md:290-292 LOBPCG examples
    a = mg.SparseSymMatrix.from_coo(3, [0, 1, 2], [0, 1, 2], [1.0, 2.0, 3.0])
    lobpcg_record("spec_diag123", a, np.ones(3), mg.SolverConfig(k=1), out, meta)
    ident = mg.SparseSymMatrix.from_coo(3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0])
    lobpcg_record("spec_b124", ident, np.array([1.0, 2.0, 4.0]), mg.SolverConfig(k=1), out, meta)
    # deflated solve on a mid-size Q (exercises smallest_above_null's LOBPCG branch, F12)
    g = synthetic.random_connected(np.random.default_rng(99), 700, extra=900, weighted=True)
    out["rand700/graph_ptr"], out["rand700/graph_idx"], out["rand700/graph_w"] = g[1], g[2], g[3]
    out["rand700/graph_n"] = np.int64(g[0])
    rec = pair_record("rand700/pair", g, out, meta)
    G = ref_graph(g)
    q = mg.two_hop_laplacian(mg.two_hop_sets(G))
    n = q.n
    cfg = mg.SolverConfig(k=8, tol=1e-6, max_iter=60, seed=42)
    lobpcg_record("rand700/q_defl", q, np.ones(n), cfg, out, meta, deflate=np.full(n, 1 / np.sqrt(n)))
    rec["eps_from_lobpcg"] = True
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def make_config(name, solve_iters=None, tight=False):
    c = synthetic.CONFIGS[name]
    t0 = time.perf_counter()
    g = synthetic.config_graph(name)
    t_graph = time.perf_counter() - t0
    out, meta = {}, {}
    n, ptr, idx, w = g
    meta["graph"] = {"n": n, "nnz": int(idx.size), "sha_indptr": sha(ptr),
                     "sha_indices": sha(idx), "sha_weights": sha(w), "seconds": t_graph}
    G = ref_graph(g)
    t0 = time.perf_counter()
    pair = mg.build_operator_pair(G)
    t_pair = time.perf_counter() - t0
    t = mg.two_hop_sets(G)
    meta["pair"] = {"eps": float(pair.epsilon), "mu": float(pair.mu),
                    "diagnostics": pair.diagnostics(), "seconds": t_pair,
                    "generalized_degree": float(pair.B.generalized_degree),
                    "A_nnz": pair.A.nnz, "Q_nnz": pair.Q.nnz, "T_nnz": int(t.indices.size),
                    "sha_A_ptr": sha(pair.A.indptr), "sha_A_idx": sha(pair.A.indices),
                    "sha_A_val": sha(pair.A.data),
                    "sha_Q_ptr": sha(pair.Q.indptr), "sha_Q_idx": sha(pair.Q.indices),
                    "sha_Q_val": sha(pair.Q.data),
                    "sha_T_ptr": sha(t.indptr), "sha_T_idx": sha(t.indices)}
    out["b"] = pair.B.b
    if n <= 5000:
        out["graph_ptr"], out["graph_idx"], out["graph_w"] = ptr, idx, w
        out["A_ptr"], out["A_idx"], out["A_val"] = pair.A.indptr, pair.A.indices, pair.A.data
        out["Q_ptr"], out["Q_idx"], out["Q_val"] = pair.Q.indptr, pair.Q.indices, pair.Q.data
    iters = c.max_iter if solve_iters is None else solve_iters
    cfg = mg.SolverConfig(k=c.k + 1, tol=c.tol, max_iter=iters, seed=42)
    t0 = time.perf_counter()
    res = mg.lobpcg_smallest(pair.A, pair.B, cfg)
    t_solve = time.perf_counter() - t0
    out["eigenvalues"] = res.eigenvalues
    out["eigenvectors"] = res.eigenvectors if n <= 5000 else res.eigenvectors.astype(np.float32)
    out["residual_norms"] = res.residual_norms
    out["converged"] = res.converged
    out["history"] = np.asarray(res.ritz_sum_history)
    meta["solve"] = {"iterations": int(res.iterations), "k": cfg.k, "tol": cfg.tol,
                     "max_iter": cfg.max_iter, "seconds": t_solve,
                     "converged": [bool(v) for v in res.converged]}
    if tight:
        import scipy.sparse.linalg as sla
        import scipy.sparse as sp
        t0 = time.perf_counter()
        w_, v_ = sla.eigsh(pair.A._csr, k=c.k + 1, M=sp.diags(pair.B.b), sigma=0.0, which="LM")
        order = np.argsort(w_)
        out["tight_eigenvalues"] = w_[order]
        meta["tight"] = {"method": "scipy eigsh shift-invert sigma=0", "seconds": time.perf_counter() - t0}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, json.dumps(meta)[:2000])


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("small", "all"):
        make_small()
    if what in ("c1", "all"):
        make_config("c1", tight=True)
    if what in ("c2", "all"):
        make_config("c2", tight=True)
