"""Full-size result check: fp64 residuals and B-orthonormality of one embed.

    python tools/check_quality.py [--config c5] [--n N] > profiles/r1_quality_c5_20M.json

Runs the solver exactly as bench.py does (same config, seed and tolerance),
then re-forms the operator pair and evaluates, in fp64 on the device (torch
CSR SpMM, not this package's kernels):
  * per column  ||A v - lambda b.v|| / ((||A||_F / sqrt(N) + |lambda| max b) ||v||),
    the quantity the reference's convergence test bounds by tol (eigensolver.py:217-222);
  * max |V' diag(b) V - I|.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--n", type=int, default=None)
    args = ap.parse_args()
    import torch
    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import core, synthetic
    cfg = synthetic.CONFIGS[args.config]
    n, ptr, idx, w = synthetic.config_graph(cfg.name, n=args.n)
    K = cfg.k
    scfg = mg.SolverConfig(k=K + 1, tol=cfg.tol, max_iter=cfg.max_iter, seed=42,
                           precision=cfg.precision)
    t0 = time.perf_counter()
    res, b, dg = core.embed_arrays(n, ptr, idx, w, K, scfg,
                                   check_connected=cfg.name != "c4")
    torch.cuda.synchronize()
    t_embed = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    V = torch.as_tensor(res.eigenvectors, device=dev).to(torch.float64)
    bv = torch.as_tensor(b, device=dev).to(torch.float64)
    lam = torch.as_tensor(res.eigenvalues, device=dev, dtype=torch.float64)

    pair = mg.build_operator_pair(mg.Graph(n, ptr, idx, w))
    A = pair.A
    Ad = torch.sparse_csr_tensor(torch.from_numpy(A.indptr).to(dev),
                                 torch.from_numpy(A.indices).to(dev),
                                 torch.from_numpy(A.data).to(dev), size=(n, n))
    AV = Ad @ V
    R = AV - (bv[:, None] * V) * lam[None, :]
    anorm = float(np.sqrt(np.sum(A.data ** 2)) / np.sqrt(n))
    vn = torch.linalg.vector_norm(V, dim=0)
    scale = (anorm + lam.abs() * bv.max()) * vn
    rel = (torch.linalg.vector_norm(R, dim=0) / scale).cpu().numpy()
    G = V.T @ (bv[:, None] * V)
    orth = float((G - torch.eye(G.shape[0], device=dev, dtype=torch.float64)).abs().max())
    out = {
        "config": cfg.name, "n": int(n), "K": K, "block": K + 1, "tol": cfg.tol,
        "precision": cfg.precision, "iterations": int(res.iterations),
        "embed_s_incl_h2d": t_embed,
        "converged": bool(np.all(res.converged)),
        "epsilon_solver": float(dg.epsilon), "epsilon_pair": float(pair.epsilon),
        "eigenvalues": [float(x) for x in res.eigenvalues],
        "fp64_relative_residuals": [float(x) for x in rel],
        "max_fp64_relative_residual": float(rel.max()),
        "max_fp64_relative_residual_over_tol": float(rel.max() / cfg.tol),
        "b_orthonormality_max_abs": orth,
        "note": "residuals re-evaluated in fp64 with torch CSR SpMM on the re-formed A "
                "(reference convergence quantity, eigensolver.py:217-222)",
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
