"""ctypes binding of the C ABI in include/manigraph_b200.h (libmgb200.so).

This is the binding a maintainer would add to the reference package (which
has no FFI of its own): plain pointers, sizes and status codes.  The library
is loaded from ``paper_2112_07862_b200/_native/libmgb200.so`` (built in-tree
by ``__graft_entry__.build()``); there is no fallback -- if the library or a
CUDA device is missing, every compute call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_native", "libmgb200.so")

MG_OK, MG_ERR_INPUT, MG_ERR_DISCONNECTED, MG_ERR_NOT_CONVERGED = 0, 1, 2, 3
MG_ERR_CUDA, MG_ERR_NCCL, MG_ERR_NOMEM, MG_ERR_INTERNAL = 4, 5, 6, 7
MG_ERR_PARSE = 8

i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p
P_i64 = C.POINTER(C.c_int64)
P_i32 = C.POINTER(C.c_int32)
P_f64 = C.POINTER(C.c_double)
P_int = C.POINTER(C.c_int)


class SolverCfg(C.Structure):
    _fields_ = [("k", i32), ("max_iter", i32), ("tol", f64), ("preconditioner", i32),
                ("precision", i32), ("reorder", i32), ("reserved", i32)]


class SolverOut(C.Structure):
    _fields_ = [("eigenvalues", P_f64), ("residual_norms", P_f64), ("converged", P_i32),
                ("history", P_f64), ("history_cap", i32), ("iterations", i32),
                ("history_len", i32), ("normals_used", i32)]


class EmbedDiag(C.Structure):
    _fields_ = [("mu", f64), ("epsilon", f64), ("min_disc_left_end", f64),
                ("dropped_eigenvalue", f64), ("generalized_degree", f64),
                ("binding_row", i64), ("q_nnz", i64), ("a_nnz", i64), ("t_nnz", i64),
                ("n_components", i64), ("iterations", i32), ("eps_iterations", i32),
                ("seconds_setup", f64), ("seconds_eps", f64), ("seconds_solve", f64),
                ("fast_steps", i64), ("fast_fallbacks", i64)]


# name -> argtypes (restype is always c_int status, except mg_last_error / mg_version)
SIGNATURES = {
    "mg_device_count": [P_int],
    "mg_ctx_create": [C.c_int, vp, C.POINTER(vp)],
    "mg_ctx_destroy": [vp],
    "mg_ctx_set_stream": [vp, vp],
    "mg_ctx_launch_count": [vp, P_i64],
    "mg_ctx_get_stream": [vp, C.POINTER(vp)],
    "mg_ctx_set_profiling": [vp, C.c_int],
    "mg_ctx_stats": [vp, P_i64, P_f64, P_f64],
    "mg_components": [vp, i64, vp, vp, vp, P_i64],
    "mg_laplacian": [vp, i64, vp, vp, vp, vp, vp, vp],
    "mg_two_hop_count": [vp, i64, vp, vp, vp, P_i64],
    "mg_two_hop_fill": [vp, i64, vp, vp, vp, vp],
    "mg_two_hop_laplacian_count": [vp, i64, vp, vp, P_i64],
    "mg_two_hop_laplacian_fill": [vp, i64, vp, vp, C.c_int, vp, vp, vp],
    "mg_check_symmetric": [vp, i64, vp, vp, vp, f64, P_int],
    "mg_repulsion_weight": [vp, i64, vp, vp, vp, f64, P_f64],
    "mg_assemble_count": [vp, i64, vp, vp, vp, vp, vp, vp, f64, f64, vp, P_i64],
    "mg_assemble_fill": [vp, i64, vp, vp, vp, vp, vp, vp, f64, f64, vp, vp, vp],
    "mg_degree_balancing": [vp, i64, vp, vp, vp, vp, P_f64, P_i64],
    "mg_disc_left_min": [vp, i64, vp, vp, vp, P_f64, P_i64],
    "mg_row_sums": [vp, i64, vp, vp, vp],
    "mg_gershgorin": [vp, i64, vp, vp, vp, vp, vp, vp],
    "mg_frobenius_norm": [vp, i64, vp, P_f64],
    "mg_balance_radii": [vp, i64, vp, vp, P_f64],
    "mg_lobpcg": [vp, i64, vp, vp, vp, vp, C.POINTER(SolverCfg), vp, i64, vp, vp,
                  C.POINTER(SolverOut)],
    "mg_lobpcg_deflate": [vp, i64, vp, vp, vp, vp, C.POINTER(SolverCfg), vp, i64, vp, i32, vp,
                          C.POINTER(SolverOut)],
    "mg_identity_shift": [vp, i64, vp, vp, vp, vp, i64, i32, P_f64],
    "mg_smallest_above_null": [vp, i64, vp, vp, vp, f64, f64, i32, vp, i64, i32, P_f64],
    "mg_spmm": [vp, i64, vp, vp, vp, vp, i32, vp],
    "mg_embed": [vp, i64, vp, vp, vp, i32, C.POINTER(SolverCfg), i32, i32, i32, vp, i64, vp, vp,
                 C.POINTER(SolverOut), C.POINTER(EmbedDiag)],
    "mg_embed_host": [vp, i64, vp, vp, vp, i32, C.POINTER(SolverCfg), i32, i32, i32, vp, i64,
                      vp, vp, C.POINTER(SolverOut), C.POINTER(EmbedDiag)],
    "mg_gram_pair_f32": [vp, i64, i32, i32, vp, vp, vp, vp, vp],
    "mg_update_f32": [vp, i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp],
    "mg_kmeans": [vp, i64, i32, vp, i32, i32, C.c_uint64, vp, P_f64],
    "mg_knn_graph_count": [vp, i64, i32, vp, i32, i32, vp, P_i64],
    "mg_normal_stream": [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, i64, vp],
    "mg_copy_d2h": [vp, vp, vp, i64],
    "mg_copy_h2d": [vp, vp, vp, i64],
    "mg_save_embedding_csv": [C.c_char_p, i64, i32, vp, i32],
    "mg_load_embedding_csv_dims": [C.c_char_p, P_i64, P_i32],
    "mg_load_embedding_csv": [C.c_char_p, i64, i32, vp, i32],
    "mg_save_edge_list": [C.c_char_p, i64, vp, vp, vp, i32],
    "mg_load_edge_list_count": [C.c_char_p, i32, P_i64, P_i64, P_i64],
    "mg_load_edge_list_fill": [vp, vp, vp],
    "mg_save_embedding_bin": [C.c_char_p, i64, i32, vp, vp, vp, C.c_char_p, i32],
    "mg_load_embedding_bin_dims": [C.c_char_p, P_i64, C.POINTER(i32), C.POINTER(i32), C.c_char_p],
    "mg_load_embedding_bin": [C.c_char_p, vp, vp, vp, i32],
    "mg_save_graph_bin": [C.c_char_p, i64, vp, vp, vp, i32],
    "mg_load_graph_bin_dims": [C.c_char_p, P_i64, P_i64],
    "mg_load_graph_bin": [C.c_char_p, vp, vp, vp, i32],
    "mg_knn_graph_fill": [vp, i64, i32, vp, i32, i32, vp, vp],
    "mg_normalize_rows": [vp, i64, i32, vp, vp],
    # multi-GPU (row-partitioned solve)
    "mg_nccl_unique_id": [vp],
    "mg_comm_create_nccl": [vp, i32, i32, vp, C.POINTER(vp)],
    "mg_local_group_create": [i32, C.POINTER(vp)],
    "mg_local_group_destroy": [vp],
    "mg_comm_create_local": [vp, i32, C.POINTER(vp)],
    "mg_comm_destroy": [vp],
    "mg_embed_dist": [vp, vp, i64, vp, vp, vp, i32, C.POINTER(SolverCfg), i32, i32, i32, vp, i64,
                      vp, vp, C.POINTER(SolverOut), C.POINTER(EmbedDiag)],
    "mg_dist_plan_host": [i64, vp, vp, i32, i32, C.c_void_p, vp, vp, vp, vp, vp, vp, vp],
}


class DistPlanInfo(C.Structure):
    _fields_ = [("r0", i64), ("nloc", i64), ("nhalo", i64), ("nsend", i64), ("local_nnz", i64)]


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing (there is no CPU path)."""


class NativeError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the native library (no CUDA calls are made)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"native library not built: {path} (run __graft_entry__.build())")
        lib = C.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.mg_last_error.restype = C.c_char_p
        lib.mg_last_error.argtypes = []
        lib.mg_version.restype = C.c_int
        lib.mg_version.argtypes = []
        _lib = lib
        return lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != MG_OK:
        msg = lib.mg_last_error().decode("utf-8", "replace")
        raise NativeError(rc, msg)
    return rc


_ctx = {}


def context(device: int = 0):
    """Process-wide library context on ``device`` (library-owned stream)."""
    if device in _ctx:
        return _ctx[device]
    lib = load()
    n = C.c_int(0)
    rc = lib.mg_device_count(C.byref(n))
    if rc != MG_OK or n.value <= device:
        raise NativeUnavailable("no CUDA device available for the sm_100a path: "
                                + lib.mg_last_error().decode())
    h = vp()
    call("mg_ctx_create", device, None, C.byref(h))
    _ctx[device] = h
    return h


PROF_CLASSES = ("spmm", "gram", "update", "resid", "ctrl", "setup")


def stream_handle(device: int = 0) -> int:
    h = vp()
    call("mg_ctx_get_stream", context(device), C.byref(h))
    return int(h.value or 0)


def set_profiling(enable: bool, device: int = 0):
    call("mg_ctx_set_profiling", context(device), int(bool(enable)))


def stats(device: int = 0) -> dict:
    import numpy as np
    cnt = np.zeros(6, np.int64)
    ms = np.zeros(6)
    by = np.zeros(6)
    call("mg_ctx_stats", context(device), cnt.ctypes.data_as(P_i64), ms.ctypes.data_as(P_f64),
         by.ctypes.data_as(P_f64))
    return {name: {"launches": int(cnt[i]), "ms": float(ms[i]), "bytes": float(by[i])}
            for i, name in enumerate(PROF_CLASSES)}


def launch_count(device: int = 0) -> int:
    v = C.c_int64(0)
    call("mg_ctx_launch_count", context(device), C.byref(v))
    return int(v.value)
