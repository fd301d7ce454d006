"""Standalone check and timing of mg_update_f32 (variant 0: fp32 FMA k_update_ws, 1: tcgen05).

    python tools/bench_update.py [n ...]      (MG_U3_DBG=1|2|4: timing experiments of the tcgen05 kernel)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2112_07862_b200 import _native as N  # noqa: E402


def make(n, m, mp, ld, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    S = torch.zeros(n, ld, device="cuda")
    AS = torch.zeros(n, ld, device="cuda")
    for blk, sc in ((0, 1e-3), (1, 1e-5), (2, 3e-6)):
        S[:, blk * mp:blk * mp + m] = torch.randn(n, m, device="cuda", generator=g) * sc
        AS[:, blk * mp:blk * mp + m] = torch.randn(n, m, device="cuda", generator=g) * sc * 3
    b = torch.rand(n, device="cuda", generator=g) + 0.5
    prec = 1.0 / (torch.rand(n, device="cuda", generator=g) * 20 + 5)
    w = 3 * mp
    Zp = torch.zeros(w, mp, device="cuda")
    Zp[:, :m] = torch.randn(w, m, device="cuda", generator=g) * 0.3
    Zp[:mp] *= 1e-3  # X rows of Zp: the projection part
    for blk in range(3):
        Zp[blk * mp + m:(blk + 1) * mp] = 0
    Yx = torch.zeros(mp, mp, device="cuda")
    Yx[:m, :m] = torch.eye(m, device="cuda") + torch.randn(m, m, device="cuda", generator=g) * 1e-2
    M = torch.cat([Zp.reshape(-1), Yx.reshape(-1)]).contiguous()
    theta = torch.rand(m, device="cuda", generator=g, dtype=torch.float64) * 1e-2 + 1e-3
    return S, AS, b, prec, M, theta, Zp, Yx


def reference(S, AS, b, prec, Zp, Yx, theta, m, mp):
    S64, A64 = S.double(), AS.double()
    w = 3 * mp
    P = S64[:, :w] @ Zp.double()
    AP = A64[:, :w] @ Zp.double()
    X = S64[:, :mp] @ Yx.double() + P
    AX = A64[:, :mp] @ Yx.double() + AP
    th = torch.zeros(mp, dtype=torch.float64, device="cuda")
    th[:m] = theta
    R = AX - b.double()[:, None] * X * th[None, :]
    R[:, m:] = 0
    W = prec.double()[:, None] * R
    return X, P, W, AX, AP, (R * R).sum(0), (X * X).sum(0)


def call(variant, n, ld, m, mp, S, AS, b, prec, M, theta, wc, cs):
    p = lambda t: C.c_void_p(t.data_ptr())
    torch.cuda.synchronize()  # the library runs on its own stream
    N.call("mg_update_f32", N.context(0), variant, n, ld, m, mp, p(S), p(AS), p(b), p(prec), p(M),
           p(theta), p(wc), p(cs))


def main():
    ns = [int(x) for x in sys.argv[1:]] or [200_000, 2_000_000, 20_000_000]
    m, mp, ld = 33, 36, 116
    for n in ns:
        S, AS, b, prec, M, theta, Zp, Yx = make(n, m, mp, ld)
        ref = reference(S, AS, b, prec, Zp, Yx, theta, m, mp) if n <= 2_000_000 else None
        for variant in (0, 1):
            S1, A1 = S.clone(), AS.clone()
            wc = torch.zeros(n, mp, device="cuda")
            cs = torch.zeros(2 * mp, dtype=torch.float64, device="cuda")
            call(variant, n, ld, m, mp, S1, A1, b, prec, M, theta, wc, cs)
            if ref is not None:
                X, P, W, AX, AP, sr, sx = ref
                got = (S1[:, :mp], S1[:, mp:2 * mp], S1[:, 2 * mp:3 * mp], A1[:, :mp], A1[:, mp:2 * mp])
                names = ("X", "P", "W", "AX", "AP")
                msg = []
                for nm, g_, r_ in zip(names, got, (X, P, W, AX, AP)):
                    err = (g_.double() - r_).abs().max().item()
                    msg.append(f"{nm} {err:.2e}/{r_.abs().max().item():.2e}")
                msg.append(f"Wc==W {bool((wc == S1[:, 2 * mp:3 * mp]).all())}")
                msg.append(f"sr {((cs[:mp] - sr).abs().max() / sr.abs().max()).item():.1e}")
                msg.append(f"sx {((cs[mp:] - sx).abs().max() / sx.abs().max()).item():.1e}")
                print(f"n={n} variant {variant}: max err/max | " + " ".join(msg), flush=True)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            R = 5
            torch.cuda.synchronize()
            ev[0].record()
            for _ in range(R):
                call(variant, n, ld, m, mp, S1, A1, b, prec, M, theta, wc, cs)
            ev[1].record()
            torch.cuda.synchronize()
            dt = ev[0].elapsed_time(ev[1]) / R
            print(f"n={n} variant {variant}: {dt:.3f} ms/call (incl. sync + part sums) "
                  f"{10 * mp * 4 * n / dt / 1e6:.0f} GB/s algorithmic", flush=True)
        del S, AS


if __name__ == "__main__":
    main()
