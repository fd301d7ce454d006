"""Device knn_graph (reference semantics, graph.py:281-315) at config scale.

    python tools/bench_knn.py [--config c5] [--n 20000000] [--k 8]

Prints one JSON line: seconds for the device graph (grid search, union,
sigma^2 = mean retained d^2, CSR), and for comparison the harness's host
cKDTree build of the same point cloud (synthetic.knn_csr, the config's
median-sigma rule) that bench.py uses.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--no-host", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import synthetic
    cfg = synthetic.CONFIGS[a.config]
    n = a.n or cfg.n
    k = a.k or cfg.knn
    x = synthetic.points(cfg.name, n)
    xd = torch.from_numpy(x).cuda()
    mg.knn_graph(xd[:200_000], k)  # warm-up (module load, pools)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = mg.knn_graph(xd, k)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    out = {"config": cfg.name, "n": n, "k": k, "device_s": t_dev, "edges": g.num_edges}
    if not a.no_host:
        t0 = time.perf_counter()
        synthetic.knn_csr(x, k)
        out["host_ckdtree_s"] = time.perf_counter() - t0
        out["host_cores"] = os.cpu_count()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
