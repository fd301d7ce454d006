"""Standalone timing of mg_gram_pair_f32 (MG_TC_V=1: v1 kernel, else v2). VS / NS env: versions / sizes."""
import ctypes as C, sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2112_07862_b200 import _native as N
w, ld = 108, 116
for n in [int(x) for x in os.environ.get("NS", "2000000 20000000").split()]:
    S = torch.randn(n, ld, device='cuda') / 1000
    AS = torch.randn(n, ld, device='cuda') / 1000
    b = torch.rand(n, device='cuda') + 0.5
    GB = torch.zeros(w*w, dtype=torch.float64, device='cuda'); GA = torch.zeros_like(GB)
    for v in os.environ.get('VS', '1 2').split():  # MG_TC_V value: 1 = v1, 2 = v2, else v4
        os.environ['MG_TC_V'] = v
        f = lambda: N.call("mg_gram_pair_f32", N.context(0), n, ld, w, C.c_void_p(S.data_ptr()), C.c_void_p(AS.data_ptr()),
                   C.c_void_p(b.data_ptr()), C.c_void_p(GB.data_ptr()), C.c_void_p(GA.data_ptr()))
        f(); torch.cuda.synchronize()
        t = time.perf_counter(); R = 5
        for _ in range(R): f()
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / R
        print(f"n={n} v{v}: {dt*1e3:.3f} ms/call (incl. host sync, memset, reduce)  {2*n*w*4/dt/1e9:.0f} GB/s", flush=True)
    del S, AS
