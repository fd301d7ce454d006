import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")
    config.addinivalue_line("markers", "slow: long-running (large synthetic configs)")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    return z, meta


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small")


@pytest.fixture(scope="session")
def golden_c1():
    return load_golden("c1")


@pytest.fixture(scope="session")
def golden_c2():
    return load_golden("c2")


def graph_from_golden(z, name):
    return (int(z[f"{name}/graph_n"]), z[f"{name}/graph_ptr"], z[f"{name}/graph_idx"],
            z[f"{name}/graph_w"])


def principal_angles(U, V, b=None):
    """Principal angles between span(U) and span(V) in the B inner product."""
    if b is not None:
        s = np.sqrt(np.asarray(b, np.float64))[:, None]
        U, V = U * s, V * s
    qu, _ = np.linalg.qr(U)
    qv, _ = np.linalg.qr(V)
    sv = np.linalg.svd(qu.T @ qv, compute_uv=False)
    sv = np.clip(sv, -1.0, 1.0)
    # arcsin of the sine form is accurate for tiny angles
    m = qv - qu @ (qu.T @ qv)
    ss = np.linalg.svd(m, compute_uv=False)
    return np.arcsin(np.clip(np.sort(ss)[::-1], 0.0, 1.0))


def clusters(vals, rel_gap):
    """Split sorted eigenvalues into maximal runs with relative gaps < rel_gap."""
    out, cur = [], [0]
    for i in range(1, len(vals)):
        scale = max(abs(vals[i]), abs(vals[i - 1]), 1e-300)
        if abs(vals[i] - vals[i - 1]) < rel_gap * scale:
            cur.append(i)
        else:
            out.append(cur)
            cur = [i]
    out.append(cur)
    return out
