"""tcgen05 (3xTF32) Gram pair vs an fp64 numpy Gram of the same fp32 data.

3xTF32 products carry ~2^-21 relative error and the MMA accumulates 128 rows
in fp32 before the fp64-accurate fold, so the bar is 2e-6 of the Gram's scale
(sum of |products|), tighter than the fp32 data's own 6e-8 per element times
sqrt(rows) growth would allow for plain fp32 summation.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gram_tc(S, AS, b, w):
    import torch
    assert S.dtype == AS.dtype == b.dtype == np.float32
    from paper_2112_07862_b200 import _native as N
    n, ld = S.shape
    dS = torch.from_numpy(S).cuda()
    dA = torch.from_numpy(AS).cuda()
    db = torch.from_numpy(b).cuda()
    GB = torch.zeros(w * w, dtype=torch.float64, device="cuda")
    GA = torch.zeros(w * w, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    N.call("mg_gram_pair_f32", N.context(0), n, ld, w, C.c_void_p(dS.data_ptr()),
           C.c_void_p(dA.data_ptr()), C.c_void_p(db.data_ptr()), C.c_void_p(GB.data_ptr()),
           C.c_void_p(GA.data_ptr()))
    return GB.cpu().numpy().reshape(w, w), GA.cpu().numpy().reshape(w, w)


@pytest.mark.parametrize("n,w,ld", [(100_003, 108, 116), (4_099, 68, 72), (37, 100, 104), (50_001, 60, 68),
                                    (1_000_000, 108, 116)])
def test_gram_pair_tc_vs_fp64(n, w, ld):
    bar = 2e-6
    rng = np.random.default_rng(n)
    S = rng.standard_normal((n, ld)) / np.sqrt(n)
    S[:, :8] *= 40.0          # mixed column scales (X vs W blocks)
    S = S.astype(np.float32)
    AS = (rng.standard_normal((n, ld)) * 0.3 / np.sqrt(n)).astype(np.float32)
    b = rng.uniform(0.5, 2.0, n).astype(np.float32)
    GB, GA = _gram_tc(S, AS, b, w)
    S64, A64, b64 = S[:, :w].astype(np.float64), AS[:, :w].astype(np.float64), b.astype(np.float64)
    bS = (b[:, None] * S[:, :w]).astype(np.float32).astype(np.float64)  # the kernel scales in fp32
    # block-lower 8x8 blocks are mirrored from the block-upper products
    # (S'AS is symmetric for symmetric A; here AS is random)
    def sym(M):
        out = M.copy()
        I, J = np.indices(M.shape)
        low = (I >> 3) > (J >> 3)
        out[low] = M.T[low]
        return out
    RB = sym(S64.T @ bS)
    RA = sym(S64.T @ A64)
    scaleB = sym(np.abs(S64).T @ np.abs(bS))
    scaleA = sym(np.abs(S64).T @ np.abs(A64))
    eb, ea = np.max(np.abs(GB - RB) / scaleB), np.max(np.abs(GA - RA) / scaleA)
    print("rel err", eb, ea)
    assert eb < bar and ea < bar
    I, J = np.indices(GB.shape)
    low = (I >> 3) > (J >> 3)
    np.testing.assert_array_equal(GB[low], GB.T[low])
    np.testing.assert_array_equal(GA[low], GA.T[low])
