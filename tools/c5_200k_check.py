import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, json
sys.path.insert(0, '/root/repo/tests')
import paper_2112_07862_b200 as mg
from paper_2112_07862_b200 import core, synthetic
import importlib.util
spec = importlib.util.spec_from_file_location("tsp", "/root/repo/tests/test_gpu_scale_parity.py")
tsp = importlib.util.module_from_spec(spec); spec.loader.exec_module(tsp)
z, meta = tsp.load("c5_200K")
c = synthetic.CONFIGS[meta["config"]]
g = tsp.graph("c5_200K", meta)
seed = int(os.environ.get("SEED", "42"))
cfg = mg.SolverConfig(k=c.k + 1, tol=c.tol, max_iter=3000, seed=seed, precision="fp32")
res, bt, dg = core.embed_arrays(*g, c.k, cfg)
tight = z["tight_eigenvalues"][:c.k + 1]; ref = z["ref_eigenvalues"]
rel = np.abs(res.eigenvalues - tight) / tight
print("seed", seed, "iterations", res.iterations, "conv", bool(res.converged.all()), "max rel_t first29 %.2e last4 %s" % (rel[:29].max(), np.array2string(rel[-4:], precision=1)), "resid last4", np.array2string(np.asarray(res.residual_norms[-4:]), precision=1))

vecs = res.eigenvectors.cpu().numpy(); b = bt.cpu().numpy()
V = z["tight_eigenvectors"].astype(np.float64)
out = []
for cl, ra in zip(meta["clusters"]["complete"], meta["clusters"]["ref_angle_per_cluster"]):
    ang = float(tsp.principal_angles(vecs[:, cl], V[:, cl], b).max())
    out.append("%.1f" % (ang / ra))
print("angle / reference angle per complete cluster:", " ".join(out))
