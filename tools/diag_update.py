import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tools.bench_update import make, reference, call
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
m, mp, ld = 33, 36, 116
S, AS, b, prec, M, theta, Zp, Yx = make(n, m, mp, ld)
ref = reference(S, AS, b, prec, Zp, Yx, theta, m, mp)
for rep in range(2):
    S1, A1 = S.clone(), AS.clone()
    wc = torch.zeros(n, mp, device="cuda"); cs = torch.zeros(2 * mp, dtype=torch.float64, device="cuda")
    call(1, n, ld, m, mp, S1, A1, b, prec, M, theta, wc, cs)
    for nm, got, r in (("X", S1[:, :mp], ref[0]), ("P", S1[:, mp:2*mp], ref[1]), ("W", S1[:, 2*mp:3*mp], ref[2]),
                       ("AX", A1[:, :mp], ref[3]), ("AP", A1[:, mp:2*mp], ref[4]), ("Wc", wc, ref[2])):
        bad = ((got.double() - r).abs() > 1e-5 * r.abs().max()) | ~torch.isfinite(got)
        rows = bad.any(1).nonzero().flatten()
        cols = bad.any(0).nonzero().flatten()
        print(rep, nm, "bad rows", rows.numel(), "first", rows[:12].tolist(), "tiles", sorted(set((rows // 128).tolist()))[:10],
              "row%128", sorted(set((rows % 128).tolist()))[:20], "cols", cols.tolist()[:40], flush=True)
