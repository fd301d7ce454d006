import os, sys, json
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2112_07862_b200 as mg
from paper_2112_07862_b200 import core, synthetic
g = synthetic.config_graph("c2")
meta = json.load(open('/root/repo/tests/golden/c2.json'))
print('reference iterations', meta['solve']['iterations'])
for reorder in ['0', '1']:
    os.environ['MG_REORDER'] = reorder
    for prec in ['fp64', 'fp32']:
        cfg = mg.SolverConfig(k=5, tol=1e-6, max_iter=3000, seed=42, precision=prec)
        res, b, dg = core.embed_arrays(*g, 4, cfg)
        print('reorder', reorder, prec, 'iterations', res.iterations)
