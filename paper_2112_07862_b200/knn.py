"""Device kNN graph: drop-in for ``knn_graph`` (reference ``graph.py:281-315``).

Same arguments, errors and output (a canonical ``Graph``); the pairwise
distances, neighbour selection, union, bandwidth and CSR assembly run in
``csrc/mg_knn.cu`` (exact all-pairs search, O(n^2 d) like the reference).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .core import Graph, _call, _ctx, _dev, _empty, _ptr, _sync, _t
from .errors import InputError


def knn_graph(X, k: int, weighted: bool = True) -> Graph:
    """Symmetrized k-nearest-neighbour graph of a point cloud (graph.py:281-315)."""
    torch = _t()
    if isinstance(X, torch.Tensor):
        x = X.to(device="cuda", dtype=torch.float64)
        if x.ndim != 2:
            raise InputError("feature matrix must be 2-D")
        x = x.contiguous()
    else:
        xa = np.asarray(X, dtype=np.float64)
        if xa.ndim != 2:
            raise InputError("feature matrix must be 2-D")
        x = _dev(np.ascontiguousarray(xa), torch.float64).view(xa.shape[0], xa.shape[1])
    n, d = int(x.shape[0]), int(x.shape[1])
    k = int(k)
    if not 1 <= k < n:
        raise InputError(f"k must satisfy 1 <= k < n, got k={k}, n={n}")
    ptr = _empty(n + 1, torch.int64)
    nnz = C.c_int64(0)
    _sync()
    _call("mg_knn_graph_count", _ctx(), n, d, _ptr(x), k, int(bool(weighted)), _ptr(ptr),
          C.byref(nnz))
    idx = _empty(nnz.value, torch.int64)
    w = _empty(nnz.value, torch.float64)
    _call("mg_knn_graph_fill", _ctx(), n, d, _ptr(x), k, int(bool(weighted)), _ptr(idx), _ptr(w))
    m = nnz.value
    return Graph(n, ptr[:n + 1].cpu().numpy(), idx[:m].cpu().numpy(), w[:m].cpu().numpy())
