"""One device-resident embed of a config graph (for ncu launch lists / captures).

    python tools/prof_embed.py [--config c5] [--n 2000000] [--reps 1]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--max-iter", type=int, default=None)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--k", type=int, default=0, help="embedding dimension (default: the config's)")
    ap.add_argument("--stats", action="store_true", help="per-class CUDA-event kernel times")
    ap.add_argument("--morton", action="store_true",
                    help="experiment: number the points in Morton order of their coordinates "
                         "and skip the solver's CM reordering (MG_REORDER=0)")
    args = ap.parse_args()
    import torch
    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import core, synthetic
    cfg = synthetic.CONFIGS[args.config]
    if args.morton:
        x = synthetic.points(cfg.name, args.n)
        q = np.minimum((x - x.min(0)) / (np.ptp(x, 0) + 1e-300) * 1024, 1023).astype(np.int64)
        key = np.zeros(len(x), np.int64)
        for bit in range(10):
            for d in range(x.shape[1]):
                key |= ((q[:, d] >> bit) & 1) << (x.shape[1] * bit + d)
        x = x[np.argsort(key, kind="stable")]
        n, ptr, idx, w = synthetic.knn_csr(x, cfg.knn)
        import os
        os.environ["MG_REORDER"] = "0"
    else:
        n, ptr, idx, w = synthetic.config_graph(cfg.name, n=args.n)
    K = args.k or cfg.k
    scfg = mg.SolverConfig(k=K + 1, tol=cfg.tol, max_iter=args.max_iter or cfg.max_iter, seed=args.seed,
                           precision=cfg.precision)
    zh = np.random.default_rng(args.seed).standard_normal(core._stream_size(n, max(K + 1, 8)))
    dd = torch.device("cuda", 0)
    dev = (torch.from_numpy(np.ascontiguousarray(ptr, np.int64)).to(dd),
           torch.from_numpy(np.ascontiguousarray(idx, np.int64)).to(dd),
           torch.from_numpy(np.ascontiguousarray(w, np.float64)).to(dd), torch.from_numpy(zh).to(dd))
    from paper_2112_07862_b200 import _native as N
    for r in range(args.reps):
        if args.stats and r == args.reps - 1:
            N.set_profiling(True, 0)
            N.stats(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, b, dg = core.embed_arrays(n, None, None, None, K, scfg, device_inputs=dev)
        torch.cuda.synchronize()
        print(f"rep {r}: {time.perf_counter() - t0:.3f} s, iterations {res.iterations}, "
              f"eps_it {dg.eps_iterations}, ev[:4] {np.asarray(res.eigenvalues)[:4]}, "
              f"setup {dg.seconds_setup:.3f} eps {dg.seconds_eps:.3f} solve {dg.seconds_solve:.3f}", flush=True)
    if args.stats:
        st = N.stats(0)
        N.set_profiling(False, 0)
        for k, v in st.items():
            if v["launches"]:
                print(f"  {k:8s} {v['launches']:6d} launches {v['ms']:9.1f} ms "
                      f"{1e3 * v['ms'] / v['launches']:9.1f} us/launch "
                      f"{v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
