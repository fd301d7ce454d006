"""Host logic of the row-partitioned solve, no GPU needed.

``mg_dist_plan_host`` is the planner the device build (mg_dist.cu) uses: row
ranges, sorted halo rows, per-peer receive/send slots and the remapped local
CSR.  Checked here (1) for internal consistency over every rank pair and
(2) end to end over a real 2-process ``gloo`` group: halo rows travel by
send/recv exactly as the plan says, the local SpMM equals the matching rows of
the global SpMM, and allreduced local Gram blocks equal the global Gram.
"""

import os
import socket

import numpy as np
import pytest

from paper_2112_07862_b200 import dist, synthetic


def _graphs():
    rng = np.random.default_rng(11)
    yield "tree+extra", synthetic.random_connected(rng, 400, extra=300, weighted=True)
    yield "path", synthetic.from_edges(50, np.arange(49), np.arange(1, 50), np.ones(49))
    yield "tiny", synthetic.from_edges(3, [0, 1], [1, 2], [1.0, 2.0])


def _spmm(ptr, idx, w, X):
    Y = np.zeros((ptr.size - 1, X.shape[1]))
    for r in range(ptr.size - 1):
        s, e = ptr[r], ptr[r + 1]
        Y[r] = w[s:e] @ X[idx[s:e]]
    return Y


def _local_spmm(p, w_local, X_ext):
    return _spmm(p["local_indptr"], p["local_indices"], w_local, X_ext)


@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_plan_consistency_and_local_spmm(R):
    for name, (n, ptr, idx, w) in _graphs():
        plans = [dist.plan(ptr, idx, R, r) for r in range(R)]
        # row ranges tile [0, n)
        assert plans[0]["r0"] == 0
        assert sum(p["nloc"] for p in plans) == n
        for a, b in zip(plans, plans[1:]):
            assert b["r0"] == a["r0"] + a["nloc"]
        X = np.random.default_rng(3).standard_normal((n, 5))
        Y = _spmm(ptr, idx, w, X)
        for me, p in enumerate(plans):
            r0, nl = p["r0"], p["nloc"]
            halo = p["halo"]
            assert np.all(np.diff(halo) > 0), name           # sorted, unique
            assert np.all((halo < r0) | (halo >= r0 + nl))   # remote only
            cols = idx[ptr[r0]:ptr[r0 + nl]]
            remote = np.unique(cols[(cols < r0) | (cols >= r0 + nl)])
            np.testing.assert_array_equal(halo, remote)
            # receive slots from peer q == q's send list to me, row for row
            for q, pq in enumerate(plans):
                if q == me:
                    assert p["rcnt"][q] == 0 and p["scnt"][q] == 0
                    continue
                assert p["rcnt"][q] == pq["scnt"][me]
                sent = pq["send_rows"][pq["soff"][me]:pq["soff"][me] + pq["scnt"][me]] + pq["r0"]
                got = halo[p["roff"][q]:p["roff"][q] + p["rcnt"][q]]
                np.testing.assert_array_equal(sent, got)
            # local SpMM on [local | halo] rows == global rows [r0, r0+nl)
            X_ext = np.concatenate([X[r0:r0 + nl], X[halo]])
            wl = w[ptr[r0]:ptr[r0 + nl]]
            np.testing.assert_array_equal(_local_spmm(p, wl, X_ext), Y[r0:r0 + nl])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        n, ptr, idx, w = synthetic.random_connected(np.random.default_rng(11), 400, extra=300,
                                                    weighted=True)
        b = np.random.default_rng(4).uniform(0.5, 2.0, n)
        p = dist.plan(ptr, idx, world, rank)
        r0, nl = p["r0"], p["nloc"]
        X = np.random.default_rng(3).standard_normal((n, 6))   # same on all ranks
        Xl = X[r0:r0 + nl]
        # halo exchange by the plan (what NcclComm::exchange does with send/recv)
        send = torch.from_numpy(np.ascontiguousarray(Xl[p["send_rows"]]))
        recv = torch.zeros((p["halo"].size, 6), dtype=torch.float64)
        reqs = []
        for peer in range(world):
            if peer == rank:
                continue
            so, sc = int(p["soff"][peer]), int(p["scnt"][peer])
            ro, rc = int(p["roff"][peer]), int(p["rcnt"][peer])
            if sc:
                reqs.append(tdist.isend(send[so:so + sc].contiguous(), peer))
            if rc:
                buf = torch.zeros((rc, 6), dtype=torch.float64)
                reqs.append((tdist.irecv(buf, peer), buf, ro))
        for rq in reqs:
            if isinstance(rq, tuple):
                rq[0].wait()
                recv[rq[2]:rq[2] + rq[1].shape[0]] = rq[1]
            else:
                rq.wait()
        X_ext = np.concatenate([Xl, recv.numpy()])
        Yl = _local_spmm(p, w[ptr[r0]:ptr[r0 + nl]], X_ext)
        Y = _spmm(ptr, idx, w, X)
        ok_spmm = bool(np.array_equal(Yl, Y[r0:r0 + nl]))
        # Gram allreduce: sum over ranks of local X^T B X == global
        G = torch.from_numpy(Xl.T @ (b[r0:r0 + nl, None] * Xl))
        tdist.all_reduce(G)
        ok_gram = bool(np.allclose(G.numpy(), X.T @ (b[:, None] * X), rtol=1e-13, atol=1e-12))
        # gathered rows reproduce the full product
        parts = [torch.zeros(1)] * world
        tdist.all_gather_object(parts, (r0, Yl))
        full = np.zeros_like(Y)
        for pr0, py in parts:
            full[pr0:pr0 + py.shape[0]] = py
        ok_full = bool(np.array_equal(full, Y))
        tdist.destroy_process_group()
        q.put((rank, ok_spmm, ok_gram, ok_full, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, False, False, repr(e)))


def test_gloo_world2_halo_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_spmm, ok_gram, ok_full, err in res:
        assert err is None, err
        assert ok_spmm and ok_gram and ok_full, (rank, ok_spmm, ok_gram, ok_full)
