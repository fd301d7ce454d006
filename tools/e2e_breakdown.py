import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2112_07862_b200 as mg
from paper_2112_07862_b200 import core, synthetic
cfg = synthetic.CONFIGS["c5"]
n, ptr, idx, w = synthetic.config_graph("c5", n=20_000_000)
K = cfg.k
scfg = mg.SolverConfig(k=K + 1, tol=cfg.tol, max_iter=cfg.max_iter, seed=42, precision=cfg.precision)
for rep in range(2):
    g = mg.Graph(n, ptr, idx, w)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev = g._device(); torch.cuda.synchronize(); t1 = time.perf_counter()
    z, nz = core._normals(scfg.seed, core._stream_size(n, max(K + 1, 8))); torch.cuda.synchronize(); t2 = time.perf_counter()
    res, b, dg = core.embed_arrays(n, None, None, None, K, scfg, device_inputs=(*dev, z)); torch.cuda.synchronize(); t3 = time.perf_counter()
    P = core._host(res.eigenvectors); t4 = time.perf_counter()
    bh = core._host(b); t5 = time.perf_counter()
    print(f"rep {rep}: H2D {t1-t0:.3f} normals {t2-t1:.3f} embed {t3-t2:.3f} D2H P {t4-t3:.3f} ({P.nbytes/1e9/(t4-t3):.1f} GB/s) D2H b {t5-t4:.3f} total {t5-t0:.3f}", flush=True)
