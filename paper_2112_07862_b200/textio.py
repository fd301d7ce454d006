"""I/O either side of the path.

Text: drop-ins for the reference's ``save_embedding_csv`` /
``load_embedding_csv`` (``embedding.py:131-166``) and ``load_edge_list`` /
``save_edge_list`` (``graph.py:147-194``): the same bytes, values and errors,
written / parsed by multi-threaded C++ (``csrc/mg_io.cu``).

Binary: ``save_embedding_bin`` / ``load_embedding_bin`` and ``save_graph_bin``
/ ``load_graph_bin`` carry the same objects (P, eigenvalues, b, method; the
canonical CSR graph) as raw arrays behind a 64-byte header
(``csrc/mg_binio.cu``), without the 17-digit text round trip.
Host-only: no GPU is needed for these.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from .errors import InputError, ParseError


def _call(name, *args, path=None, err_line=None):
    try:
        return N.call(name, *args)
    except N.NativeError as e:
        msg = str(e)
        if e.code == N.MG_ERR_PARSE and path is not None:
            prefix = f"{path}:{err_line.value}: " if err_line is not None else ""
            raise ParseError(path, err_line.value if err_line is not None else 0,
                             msg[len(prefix):] if msg.startswith(prefix) else msg) from None
        if e.code in (N.MG_ERR_INPUT, N.MG_ERR_PARSE):
            raise InputError(msg) from None
        raise


def _threads(threads):
    return int(threads) if threads else 0


def save_embedding_csv(emb, path, threads: int | None = None) -> None:
    """Write ``node,c1,...,cK`` rows with 17-significant-digit coordinates."""
    P = np.ascontiguousarray(getattr(emb, "P", emb), dtype=np.float64)
    if P.ndim != 2:
        raise InputError("embedding coordinates must be a 2-D array")
    _call("mg_save_embedding_csv", os.fsencode(path), P.shape[0], P.shape[1],
          P.ctypes.data_as(C.c_void_p), _threads(threads))


def load_embedding_csv(path, threads: int | None = None) -> np.ndarray:
    """Read coordinates written by :func:`save_embedding_csv` (rows in node order)."""
    n, k = C.c_int64(0), C.c_int32(0)
    _call("mg_load_embedding_csv_dims", os.fsencode(path), C.byref(n), C.byref(k))
    P = np.empty((n.value, k.value), dtype=np.float64)
    _call("mg_load_embedding_csv", os.fsencode(path), n.value, k.value,
          P.ctypes.data_as(C.c_void_p), _threads(threads))
    return P


def save_edge_list(g, path, threads: int | None = None) -> None:
    """Write canonical tab-separated edges (``i < j``, 17-digit weights)."""
    ptr = np.ascontiguousarray(g.indptr, dtype=np.int64)
    idx = np.ascontiguousarray(g.indices, dtype=np.int64)
    w = np.ascontiguousarray(g.weights, dtype=np.float64)
    _call("mg_save_edge_list", os.fsencode(path), int(g.n), ptr.ctypes.data_as(C.c_void_p),
          idx.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), _threads(threads))


def load_edge_list(path, threads: int | None = None):
    """Read a whitespace-separated ``i j [w]`` edge list into a canonical Graph."""
    from .core import Graph
    n, nnz, line = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    _call("mg_load_edge_list_count", os.fsencode(path), _threads(threads), C.byref(n),
          C.byref(nnz), C.byref(line), path=str(path), err_line=line)
    ptr = np.empty(n.value + 1, np.int64)
    idx = np.empty(nnz.value, np.int64)
    w = np.empty(nnz.value, np.float64)
    _call("mg_load_edge_list_fill", ptr.ctypes.data_as(C.c_void_p),
          idx.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p))
    return Graph(n.value, ptr, idx, w)


def save_embedding_bin(emb, path, threads: int | None = None) -> None:
    """Binary embedding file: P (n x K), eigenvalues, b and method of an
    ``Embedding`` (or a bare P array), bit-exact."""
    P = np.ascontiguousarray(getattr(emb, "P", emb), dtype=np.float64)
    if P.ndim != 2:
        raise InputError("embedding coordinates must be a 2-D array")
    ev = getattr(emb, "eigenvalues", None)
    ev = None if ev is None else np.ascontiguousarray(ev, dtype=np.float64)
    if ev is not None and ev.shape != (P.shape[1],):
        raise InputError("eigenvalues must have one entry per embedding column")
    b = getattr(emb, "b", None)
    b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
    if b is not None and b.shape != (P.shape[0],):
        raise InputError("b must have one entry per node")
    method = str(getattr(emb, "method", "") or "").encode()[:15]
    ptr = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _call("mg_save_embedding_bin", os.fsencode(path), P.shape[0], P.shape[1],
          P.ctypes.data_as(C.c_void_p), ptr(ev), ptr(b), method, _threads(threads))


def load_embedding_bin(path, threads: int | None = None):
    """Read a file written by :func:`save_embedding_bin` into an ``Embedding``."""
    from .core import Embedding
    n, k, hb = C.c_int64(0), C.c_int32(0), C.c_int32(0)
    method = C.create_string_buffer(16)
    _call("mg_load_embedding_bin_dims", os.fsencode(path), C.byref(n), C.byref(k), C.byref(hb),
          method, path=str(path))
    P = np.empty((n.value, k.value), dtype=np.float64)
    ev = np.empty(k.value, dtype=np.float64)
    b = np.empty(n.value, dtype=np.float64) if hb.value else None
    _call("mg_load_embedding_bin", os.fsencode(path), P.ctypes.data_as(C.c_void_p),
          ev.ctypes.data_as(C.c_void_p), None if b is None else b.ctypes.data_as(C.c_void_p),
          _threads(threads), path=str(path))
    return Embedding(P=P, method=method.value.decode(), eigenvalues=ev, b=b)


def save_graph_bin(g, path, threads: int | None = None) -> None:
    """Binary canonical-CSR graph file (indptr, indices, weights as stored)."""
    ptr = np.ascontiguousarray(g.indptr, dtype=np.int64)
    idx = np.ascontiguousarray(g.indices, dtype=np.int64)
    w = np.ascontiguousarray(g.weights, dtype=np.float64)
    _call("mg_save_graph_bin", os.fsencode(path), int(g.n), ptr.ctypes.data_as(C.c_void_p),
          idx.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), _threads(threads))


def load_graph_bin(path, threads: int | None = None):
    """Read a file written by :func:`save_graph_bin`; the CSR is checked to be the
    canonical form ``Graph.from_edges`` builds (graph.py:31-79)."""
    from .core import Graph
    n, nnz = C.c_int64(0), C.c_int64(0)
    _call("mg_load_graph_bin_dims", os.fsencode(path), C.byref(n), C.byref(nnz), path=str(path))
    ptr = np.empty(n.value + 1, np.int64)
    idx = np.empty(nnz.value, np.int64)
    w = np.empty(nnz.value, np.float64)
    _call("mg_load_graph_bin", os.fsencode(path), ptr.ctypes.data_as(C.c_void_p),
          idx.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), _threads(threads),
          path=str(path))
    return Graph(n.value, ptr, idx, w)
