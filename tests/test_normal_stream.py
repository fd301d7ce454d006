"""Device PCG64 + ziggurat normal stream vs numpy's Generator.standard_normal:
identical values (the reference's initial block, eigensolver.py:177-178)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,count", [(42, 1), (42, 4097), (0, 1_000_003), (7, 20_000_000),
                                        (2**63 + 11, 300_000)])
def test_device_stream_equals_numpy(seed, count, monkeypatch):
    monkeypatch.delenv("MG_HOST_NORMALS", raising=False)
    from paper_2112_07862_b200 import core
    z, n = core._normals(seed, count)
    ref = np.random.default_rng(seed).standard_normal(count)
    got = z.cpu().numpy()
    assert n == count
    np.testing.assert_array_equal(got, ref)
