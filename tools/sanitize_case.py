"""Small fp32 K=32 embed (C5 family, 20K nodes, a few LOBPCG iterations) so the
compute-sanitizer runs cover the wide-block kernels (tcgen05 Gram, warp-
specialised update, control step) as well as smoke()'s fp64 path.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2112_07862_b200 as mg  # noqa: E402
from paper_2112_07862_b200 import core, synthetic  # noqa: E402

n = int(os.environ.get("MG_SAN_N", "20000"))
g = synthetic.config_graph("c5", n=n)
cfg = mg.SolverConfig(k=33, tol=1e-4, max_iter=int(os.environ.get("MG_SAN_IT", "3")), seed=42,
                      precision="fp32")
res, b, dg = core.embed_arrays(*g, 32, cfg)
print("sanitize case ok: iterations", res.iterations, "eps", dg.epsilon)
