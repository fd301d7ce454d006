"""Multi-GPU embed: the LOBPCG solve row-partitioned over ranks.

The reference is single-process (numpy/scipy; eigensolver.py:165-283 runs the
whole block on one host).  Here the setup (Q, eps, mu, A, b) is replicated on
every rank -- it is a few percent of the job -- and the solve is cut into
equal row ranges of the Cuthill-McKee order: each SpMM exchanges only the halo
rows its local rows touch (NCCL grouped send/recv over NVLink/NVSwitch), and
every Gram / norm / Ritz reduction is an NCCL allreduce of a small fp64 block,
so every rank runs the identical small-matrix control sequence and ends with
the full embedding.

Two communicators:

* ``nccl_comm(rank, world, device)`` -- one process per GPU (torchrun); the
  NCCL unique id travels over the existing ``torch.distributed`` group.
* ``LocalGroup(R)`` -- R virtual ranks as threads of one process sharing one
  GPU, collectives through host memory (tests of the partitioned algorithm on
  a single B200; no kernel ever waits on another rank's kernel).

``plan()`` exposes the halo plan for a host CSR without touching a GPU (the
gloo tests use it to check the exchange logic on CPU).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N
from . import core as _core
from .core import SolverConfig, EigenResult, Embedding


class Comm:
    """Owner of an ``mg_comm`` handle."""

    def __init__(self, handle, rank: int, world: int, kind: str):
        self.handle, self.rank, self.world, self.kind = handle, rank, world, kind

    def close(self):
        if self.handle is not None:
            N.call("mg_comm_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.call("mg_nccl_unique_id", C.cast(buf, C.c_void_p))
    return bytes(buf)


def nccl_comm(rank: int, world: int, device: int, group=None) -> Comm:
    """NCCL communicator over an initialised ``torch.distributed`` group."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
    h = C.c_void_p()
    N.call("mg_comm_create_nccl", N.context(device), world, rank, C.cast(uid, C.c_void_p),
           C.byref(h))
    return Comm(h, rank, world, "nccl")


class LocalGroup:
    """R virtual ranks on one GPU (threads); ``comm(r)`` per rank."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.handle = C.c_void_p()
        N.call("mg_local_group_create", nranks, C.byref(self.handle))

    def comm(self, rank: int) -> Comm:
        h = C.c_void_p()
        N.call("mg_comm_create_local", self.handle, rank, C.byref(h))
        return Comm(h, rank, self.nranks, "local")

    def close(self):
        if self.handle:
            N.call("mg_local_group_destroy", self.handle)
            self.handle = None


def plan(indptr, indices, nranks: int, rank: int) -> dict:
    """Halo plan of ``rank`` for a host CSR (the planner the device build uses)."""
    ptr = np.ascontiguousarray(indptr, dtype=np.int64)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    n = ptr.size - 1
    info = N.DistPlanInfo()

    def vp(a):
        return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)

    N.call("mg_dist_plan_host", n, vp(ptr), vp(idx), nranks, rank, C.byref(info),
           *([C.c_void_p(0)] * 7))
    halo = np.zeros(info.nhalo, np.int64)
    roff, rcnt = np.zeros(nranks, np.int64), np.zeros(nranks, np.int64)
    soff, scnt = np.zeros(nranks, np.int64), np.zeros(nranks, np.int64)
    send = np.zeros(info.nsend, np.int32)
    lidx = np.zeros(info.local_nnz, np.int32)
    N.call("mg_dist_plan_host", n, vp(ptr), vp(idx), nranks, rank, C.byref(info), vp(halo),
           vp(roff), vp(rcnt), vp(soff), vp(scnt), vp(send), vp(lidx))
    return {"r0": int(info.r0), "nloc": int(info.nloc), "halo": halo, "roff": roff,
            "rcnt": rcnt, "soff": soff, "scnt": scnt, "send_rows": send,
            "local_indptr": ptr[info.r0:info.r0 + info.nloc + 1] - ptr[info.r0],
            "local_indices": lidx}


def embed_arrays_dist(comm: Comm, ctx, device: int, n, indptr, indices, weights, k: int,
                      cfg: SolverConfig | None = None, literal_diagonal=False,
                      check_connected=True, reorder=True, device_inputs=None):
    """Distributed ``core.embed_arrays``: every rank passes the full graph (host
    arrays, or ``device_inputs`` = (indptr, indices, weights, normals) CUDA
    tensors on ``device``) and receives the full K+1 eigenpairs, b and
    diagnostics (eigenvectors stay on the device)."""
    import torch
    dev = torch.device("cuda", device)
    cfg = cfg or SolverConfig(k=k + 1)
    s = _core._cfg_struct(cfg, k=k + 1)
    s.reserved = 1
    s.reorder = 1 if reorder else 0
    m = k + 1
    if device_inputs is None:
        p = torch.from_numpy(np.ascontiguousarray(indptr, dtype=np.int64)).to(dev)
        i = torch.from_numpy(np.ascontiguousarray(indices, dtype=np.int64)).to(dev)
        w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(dev)
        nz = _core._stream_size(n, max(m, min(8, max(n - 1, 1))))
        z = _core._normals_on(device, cfg.seed, nz, ctx)  # numpy's stream, on this GPU / context
    else:
        p, i, w, z = device_inputs
        nz = int(z.numel())
    P = torch.empty(max(n * m, 1), dtype=torch.float64, device=dev)
    b = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    ev, rn = np.zeros(m), np.zeros(m)
    cv = np.zeros(m, np.int32)
    hist = np.zeros(int(cfg.max_iter) + 2)
    out = N.SolverOut()
    out.eigenvalues = ev.ctypes.data_as(N.P_f64)
    out.residual_norms = rn.ctypes.data_as(N.P_f64)
    out.converged = cv.ctypes.data_as(N.P_i32)
    out.history = hist.ctypes.data_as(N.P_f64)
    out.history_cap = hist.size
    dg = N.EmbedDiag()
    torch.cuda.synchronize(dev)
    # A short normal stream (the eps solve doubling its block, refills) fails with the
    # same MG_ERR_INPUT on every rank: retry with a longer stream, like core.embed
    for attempt in range(4):
        try:
            N.call("mg_embed_dist", ctx, comm.handle, n, C.c_void_p(p.data_ptr()),
                   C.c_void_p(i.data_ptr()), C.c_void_p(w.data_ptr()), k, C.byref(s),
                   int(literal_diagonal), 0, int(check_connected), C.c_void_p(z.data_ptr()), nz,
                   C.c_void_p(P.data_ptr()), C.c_void_p(b.data_ptr()), C.byref(out), C.byref(dg))
            break
        except N.NativeError as e:
            if "stream exhausted" in str(e) and attempt < 3 and device_inputs is None:
                nz *= 8
                z = _core._normals_on(device, cfg.seed, nz, ctx)
                continue
            _core._raise_native(e)
    res = EigenResult(eigenvalues=ev.copy(), eigenvectors=P[:n * m].view(n, m),
                      iterations=int(out.iterations), residual_norms=rn.copy(),
                      converged=cv.astype(bool), ritz_sum_history=list(hist[:out.history_len]))
    return res, b[:n], dg


def embed_dist(comm: Comm, g, k: int, cfg: SolverConfig | None = None, device: int = 0,
               ctx=None, literal_diagonal: bool = False,
               require_convergence: bool = True) -> Embedding:
    """``embed`` (embedding.py:77-103) with the solve partitioned over ``comm``."""
    g = _core._as_graph(g)
    _core._check_k(g, k)
    ctx = ctx if ctx is not None else N.context(device)
    res, b, dg = embed_arrays_dist(comm, ctx, device, g.n, g.indptr, g.indices, g.weights, k,
                                   cfg, literal_diagonal)
    res.eigenvectors = res.eigenvectors.cpu().numpy()
    b = b.cpu().numpy()
    if require_convergence:
        _core.require_converged(res, "embedding eigensolve")
    return Embedding(P=res.eigenvectors[:, 1:], method="proposed",
                     eigenvalues=res.eigenvalues[1:], b=b,
                     diagnostics=_core._diag_dict(dg, res))


def run_local(nranks: int, fn, device: int = 0):
    """Run ``fn(comm, ctx, rank)`` on R virtual ranks (threads, one GPU each with
    its own library context/stream); returns the per-rank results."""
    group = LocalGroup(nranks)
    results, errors = [None] * nranks, [None] * nranks

    def body(r):
        h = C.c_void_p()
        comm = None
        try:
            N.call("mg_ctx_create", device, None, C.byref(h))
            comm = group.comm(r)
            results[r] = fn(comm, h, r)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors[r] = e
        finally:
            if comm is not None:
                comm.close()
            if h:
                N.call("mg_ctx_destroy", h)

    threads = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    group.close()
    for e in errors:
        if e is not None:
            raise e
    return results
