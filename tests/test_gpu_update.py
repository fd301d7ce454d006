"""The LOBPCG basis update through the C ABI (mg_update_f32), both kernels, against an fp64
restatement of eigensolver.py:255-266 on the same inputs:

    P = S Zp, X = X Yx + P, AP = AS Zp, AX = AX Yx + AP, R = AX - b X Theta, W = prec R.

variant 0 is the fp32 FMA kernel (k_update_ws).  variant 1 is the tcgen05 kernel
(k_update_tc3): it rounds the coefficient matrix Z2' = [Zp + (Yx - I) | Zp] to TF32 once and
forms only the corrections on the tensor core, so its reference uses the same rounded
coefficients (tolerance 1e-6 of each block's largest entry); against the unrounded
coefficients it is a 2^-12-inexact step in the corrections, bounded separately.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _ld(mp):
    ld = 3 * mp + 4
    return ld + 4 if (ld // 4) % 2 == 0 else ld


def _rn_tf32(x):
    """round to nearest (ties away) TF32, as the kernel rounds its coefficients"""
    i = x.contiguous().view(torch.int32)
    return ((i + 0x1000) & ~0x1FFF).view(torch.float32)


def _make(n, m, mp, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld, w = _ld(mp), 3 * mp
    S = torch.zeros(n, ld, device="cuda")
    AS = torch.zeros(n, ld, device="cuda")
    for blk, sc in ((0, 1e-3), (1, 1e-5), (2, 3e-6)):
        S[:, blk * mp:blk * mp + m] = torch.randn(n, m, device="cuda", generator=g) * sc
        AS[:, blk * mp:blk * mp + m] = torch.randn(n, m, device="cuda", generator=g) * sc * 3
    S[:, w:] = 7.0  # the deflation column / padding beyond 3mp must not leak in
    b = torch.rand(n, device="cuda", generator=g) + 0.5
    prec = 1.0 / (torch.rand(n, device="cuda", generator=g) * 20 + 5)
    Zp = torch.zeros(w, mp, device="cuda")
    Zp[:, :m] = torch.randn(w, m, device="cuda", generator=g) * 0.3
    Zp[:mp] *= 1e-3
    for blk in range(3):
        Zp[blk * mp + m:(blk + 1) * mp] = 0
    Yx = torch.zeros(mp, mp, device="cuda")
    Yx[:m, :m] = torch.eye(m, device="cuda") + torch.randn(m, m, device="cuda", generator=g) * 1e-2
    theta = torch.rand(m, device="cuda", generator=g, dtype=torch.float64) * 1e-2 + 1e-3
    return S, AS, b, prec, Zp, Yx, theta


def _reference(S, AS, b, prec, Zp, Yx, theta, m, mp, rounded):
    S64, A64, w = S.double(), AS.double(), 3 * mp
    if rounded:
        zx = Zp.clone()
        zx[:mp] += Yx - torch.eye(mp, device="cuda")
        zx, zp = _rn_tf32(zx).double(), _rn_tf32(Zp).double()
        P, AP = S64[:, :w] @ zp, A64[:, :w] @ zp
        X, AX = S64[:, :mp] + S64[:, :w] @ zx, A64[:, :mp] + A64[:, :w] @ zx
    else:
        P, AP = S64[:, :w] @ Zp.double(), A64[:, :w] @ Zp.double()
        X, AX = S64[:, :mp] @ Yx.double() + P, A64[:, :mp] @ Yx.double() + AP
    th = torch.zeros(mp, dtype=torch.float64, device="cuda")
    th[:m] = theta
    R = AX - b.double()[:, None] * X * th[None, :]
    R[:, m:] = 0
    return dict(X=X, P=P, W=prec.double()[:, None] * R, AX=AX, AP=AP, sr=(R * R).sum(0),
                sx=(X * X).sum(0))


def _call(variant, n, m, mp, S, AS, b, prec, Zp, Yx, theta):
    from paper_2112_07862_b200 import _native as N
    M = torch.cat([Zp.reshape(-1), Yx.reshape(-1)]).contiguous()
    S1, A1 = S.clone(), AS.clone()
    wc = torch.full((n, mp), 3.0, device="cuda")
    cs = torch.zeros(2 * mp, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()  # the library runs on its own stream
    p = lambda t: C.c_void_p(t.data_ptr())
    N.call("mg_update_f32", N.context(0), variant, n, _ld(mp), m, mp, p(S1), p(A1), p(b), p(prec),
           p(M), p(theta), p(wc), p(cs))
    return S1, A1, wc, cs


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("m,mp", [(33, 36), (17, 20), (9, 12)])
@pytest.mark.parametrize("n", [9973, 40000])  # a ragged last tile and whole tiles
def test_update_matches_fp64(variant, m, mp, n):
    S, AS, b, prec, Zp, Yx, theta = _make(n, m, mp, seed=mp + n)
    S1, A1, wc, cs = _call(variant, n, m, mp, S, AS, b, prec, Zp, Yx, theta)
    ref = _reference(S, AS, b, prec, Zp, Yx, theta, m, mp, rounded=variant == 1)
    got = dict(X=S1[:, :mp], P=S1[:, mp:2 * mp], W=S1[:, 2 * mp:3 * mp], AX=A1[:, :mp],
               AP=A1[:, mp:2 * mp])
    for k, v in got.items():
        err = (v.double() - ref[k]).abs().max().item()
        assert err <= 2e-6 * ref[k].abs().max().item(), (k, err)
        assert (v[:, m:] == 0).all(), k  # padding columns stay zero
    assert torch.equal(wc, got["W"])  # the compact W the SpMM reads
    assert torch.equal(S1[:, 3 * mp:], S[:, 3 * mp:])  # columns beyond 3mp untouched
    assert torch.equal(A1[:, 2 * mp:], AS[:, 2 * mp:])  # AW and beyond untouched
    assert ((cs[:mp] - ref["sr"]).abs().max() <= 1e-5 * ref["sr"].abs().max()).item()
    assert ((cs[mp:] - ref["sx"]).abs().max() <= 1e-5 * ref["sx"].abs().max()).item()


def test_tc_update_is_a_small_perturbation_of_the_exact_step():
    """Against the unrounded coefficients the tensor-core update differs by the TF32 rounding
    of the CORRECTION coefficients only: <= 2^-11 of |S| |Z2'| per entry, far below that here."""
    n, m, mp = 20000, 33, 36
    S, AS, b, prec, Zp, Yx, theta = _make(n, m, mp, seed=5)
    S1, A1, _, _ = _call(1, n, m, mp, S, AS, b, prec, Zp, Yx, theta)
    ref = _reference(S, AS, b, prec, Zp, Yx, theta, m, mp, rounded=False)
    zx = Zp.clone()
    zx[:mp] += Yx - torch.eye(mp, device="cuda")
    bound = 2.0 ** -11 * (S[:, :3 * mp].abs().double() @ zx.abs().double())
    assert ((S1[:, :mp].double() - ref["X"]).abs() <= bound + 1e-12).all()
    # and the big term X itself is carried exactly: a zero correction leaves X bit-identical
    Z0 = torch.zeros_like(Zp)
    I = torch.zeros_like(Yx)
    I[:m, :m] = torch.eye(m, device="cuda")
    S2, A2, _, _ = _call(1, n, m, mp, S, AS, b, prec, Z0, I, theta)
    assert torch.equal(S2[:, :mp], S[:, :mp]) and torch.equal(A2[:, :mp], AS[:, :mp])
