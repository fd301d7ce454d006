"""Device k-means and normalize_rows: drop-in for the C4 readout
(reference ``manigraph/clustering.py:50-134``, seeding streams ``rng.py``).

Same signatures and errors as the reference; the arithmetic runs in
``csrc/mg_kmeans.cu`` (k-means++ seeding from the reference's xoshiro256**
streams, Lloyd with the reference's empty-cluster repair, best of
``restarts``).  ``threads`` is accepted for signature compatibility (the
reference maps restarts over a thread pool, ``parallel.py``); restarts run in
sequence on the GPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import _call, _ctx, _dev, _empty, _ptr, _sync, _t
from .errors import InputError


def _coerce_points(x):
    """clustering.py:41-47: embedding objects expose their coordinates as .P."""
    src = getattr(x, "P", x)
    torch = _t()
    if isinstance(src, torch.Tensor):
        pts = src.to(device="cuda", dtype=torch.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        if pts.ndim != 2 or pts.shape[0] == 0:
            raise InputError("points must form a non-empty 2-D array")
        return pts.contiguous()
    pts = np.asarray(src, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise InputError("points must form a non-empty 2-D array")
    return _dev(np.ascontiguousarray(pts), torch.float64).view(pts.shape[0], pts.shape[1])


def normalize_rows(points) -> np.ndarray:
    """Scale each row to unit Euclidean length; zero rows stay zero (clustering.py:50-56)."""
    x = _coerce_points(points)
    n, d = x.shape
    y = _empty(n * d, _t().float64)
    _sync()
    _call("mg_normalize_rows", _ctx(), n, d, _ptr(x), _ptr(y))
    return y[:n * d].view(n, d).cpu().numpy()


def kmeans(points, c: int, restarts: int = 20, seed: int = 42, threads: int | None = None,
           return_wcss: bool = False):
    """Cluster rows of ``points`` into ``c`` groups (clustering.py:99-134).

    Deterministic for a given (seed, restarts): restart r draws from
    stream_seed(seed, r); the lowest within-cluster sum of squares wins, ties
    by the lowest restart index."""
    x = _coerce_points(points)
    n, d = x.shape
    c, restarts = int(c), int(restarts)
    if not 1 <= c <= n:
        raise InputError(f"cluster count must be in [1, {n}], got {c}")
    if restarts < 1:
        raise InputError(f"restarts must be >= 1, got {restarts}")
    lab = _empty(n, _t().int64)
    wcss = C.c_double(0.0)
    _sync()
    _call("mg_kmeans", _ctx(), n, d, _ptr(x), c, restarts, C.c_uint64(int(seed) & (2**64 - 1)),
          _ptr(lab), C.byref(wcss))
    out = lab[:n].cpu().numpy().astype(np.int64)
    return (out, float(wcss.value)) if return_wcss else out
