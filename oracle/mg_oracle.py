"""numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE).

Every function cites the reference ``file:line`` (paths relative to
``/root/reference/pkg/src/manigraph/``) whose arithmetic it restates.  The
restatement keeps the *order of floating-point operations* the reference
uses wherever the result is compared bit-exactly (sequential ``bincount``
row sums, ``(L - mu*Q) + eps*I`` with separate roundings, pairwise ``mean``),
because the CUDA path is checked against these values bit for bit.

Where the arithmetic lives in third-party code (scipy 1.18.1 ``sparsetools``
SpGEMM / CSR binops, numpy 2.3.5 + OpenBLAS 0.3.30 ``eigh``, numpy ``PCG64``
``standard_normal``) the oracle calls the same library operation; those are
the effective pins (``pyproject.toml:11-16`` only sets lower bounds).

Parity pin: ``tests/test_oracle_golden.py`` checks every function here
against ``tests/golden/*.npz``, which ``tests/golden/make_golden.py`` made by
running the unmodified reference.  Nothing here is on the product path.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "OracleInputError", "OracleDisconnected", "OracleConvergence",
    "CSR", "degrees", "laplacian", "components", "two_hop", "q_matrix",
    "check_symmetric", "identity_shift", "repulsion_weight", "assemble",
    "gershgorin_radii", "balance_radii", "degree_balancing", "operator_pair",
    "pair_diagnostics", "lobpcg", "smallest_above_null", "embed",
    "laplacian_eigenmaps", "dense_generalized_eigh", "initial_block",
    "Xoshiro256", "stream_seed", "normalize_rows", "kmeans", "knn_graph",
]

DROP_REL = 1e-12          # eigensolver.py:29
DENSE_EPS_MAX_N = 512     # operators.py:150 / eigensolver.py:446


class OracleInputError(ValueError):
    """Mirrors ``InputError`` (errors.py:10-11)."""


class OracleDisconnected(ValueError):
    """Mirrors ``DisconnectedGraphError`` (errors.py:23-32)."""

    def __init__(self, msg, n_components=None):
        super().__init__(msg)
        self.n_components = n_components


class OracleConvergence(RuntimeError):
    """Mirrors ``ConvergenceError`` (errors.py:35-45)."""

    def __init__(self, msg, result=None):
        super().__init__(msg)
        self.result = result


class CSR:
    """Plain (n, indptr, indices, data) triple; int64 indices, f64 data."""

    __slots__ = ("n", "indptr", "indices", "data")

    def __init__(self, n, indptr, indices, data):
        self.n = int(n)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.data = np.ascontiguousarray(data, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.indices.size)

    def rows(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.indptr))

    def scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.data, self.indices, self.indptr),
                             shape=(self.n, self.n))

    def diagonal(self):
        out = np.zeros(self.n)
        r = self.rows()
        on = r == self.indices
        out[r[on]] = self.data[on]
        return out

    def row_sums(self):
        # sparse.py:79-82 -- np.bincount accumulates sequentially in stored order
        return np.bincount(self.rows(), weights=self.data, minlength=self.n)

    def dense(self):
        d = np.zeros((self.n, self.n))
        d[self.rows(), self.indices] = self.data
        return d

    def matmat(self, x):
        # sparse.py:67-68 (scipy csr_matvecs)
        return self.scipy() @ x

    def frobenius(self):
        # sparse.py:76-77
        return float(np.sqrt(np.sum(self.data * self.data)))


# -- graph-level pieces ----------------------------------------------------------

def degrees(n, indptr, weights):
    """graph.py:93-96: weighted degree, sequential sum in neighbour order."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    return np.bincount(rows, weights=np.asarray(weights, np.float64), minlength=n)


def laplacian(n, indptr, indices, weights):
    """graph.py:321-346: L = D - W, diagonal stored at its sorted position."""
    indptr = np.asarray(indptr, np.int64)
    indices = np.asarray(indices, np.int64)
    weights = np.asarray(weights, np.float64)
    deg = degrees(n, indptr, weights)
    out_ptr = indptr + np.arange(n + 1, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    k_in_row = np.arange(indices.size, dtype=np.int64) - indptr[rows]
    shift = (indices > rows).astype(np.int64)          # after the diagonal slot
    pos = out_ptr[rows] + k_in_row + shift
    below = np.bincount(rows[indices < rows], minlength=n).astype(np.int64)
    dpos = out_ptr[:-1] + below
    cols = np.empty(out_ptr[-1], np.int64)
    vals = np.empty(out_ptr[-1], np.float64)
    cols[pos] = indices
    vals[pos] = -weights
    cols[dpos] = np.arange(n)
    vals[dpos] = deg
    return CSR(n, out_ptr, cols, vals)


def components(n, indptr, indices):
    """graph.py:107-123 semantics: count, labels numbered by first node seen.

    Labels from a DFS scan over s = 0..n-1 are ordered by each component's
    smallest node id; scipy's labelling is renumbered to that order.
    """
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    if n == 0:
        return 0, np.zeros(0, np.int64)
    adj = sp.csr_matrix((np.ones(len(indices)), indices, indptr), shape=(n, n))
    count, lab = connected_components(adj, directed=False)
    first = np.full(count, n, np.int64)
    np.minimum.at(first, lab, np.arange(n))
    rank = np.empty(count, np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(count)
    return int(count), rank[lab]


def two_hop(n, indptr, indices):
    """operators.py:88-108: pattern(adj @ adj) minus diagonal minus adj.

    Restated without SpGEMM: expand every path i - m - j, key it as i*n + j,
    unique (sorted), then drop i == j and the one-hop keys.
    """
    indptr = np.asarray(indptr, np.int64)
    indices = np.asarray(indices, np.int64)
    deg = np.diff(indptr)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)        # i of edge (i, m)
    cnt = deg[indices]                                        # |N(m)|
    total = int(cnt.sum())
    i_of = np.repeat(src, cnt)
    base = np.repeat(indptr[indices], cnt)
    run0 = np.repeat(np.cumsum(cnt) - cnt, cnt)
    j_of = indices[base + (np.arange(total, dtype=np.int64) - run0)]
    keys = np.unique(i_of * n + j_of)
    ii, jj = keys // n, keys % n
    keys = keys[ii != jj]
    one_hop = src * n + indices                               # already sorted
    keep = ~np.isin(keys, one_hop, assume_unique=True)
    keys = keys[keep]
    rows, cols = keys // n, keys % n
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return ptr, cols


def q_matrix(n, t_ptr, t_idx, literal_diagonal=False):
    """operators.py:111-135: Laplacian of the two-hop graph, w_ij = 1/T_i + 1/T_j."""
    t_ptr = np.asarray(t_ptr, np.int64)
    t_idx = np.asarray(t_idx, np.int64)
    counts = np.diff(t_ptr).astype(np.float64)
    inv = np.zeros(n)
    inv[counts > 0] = 1.0 / counts[counts > 0]
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(t_ptr))
    off = -(inv[rows] + inv[t_idx])
    if literal_diagonal:
        diag = inv + np.bincount(rows, weights=inv[t_idx], minlength=n)
    else:
        diag = np.bincount(rows, weights=-off, minlength=n)
    # merge the diagonal into each sorted row, then drop exact zeros
    out_ptr = t_ptr + np.arange(n + 1, dtype=np.int64)
    k_in_row = np.arange(t_idx.size, dtype=np.int64) - t_ptr[rows]
    pos = out_ptr[rows] + k_in_row + (t_idx > rows)
    below = np.bincount(rows[t_idx < rows], minlength=n).astype(np.int64)
    dpos = out_ptr[:-1] + below
    cols = np.empty(out_ptr[-1], np.int64)
    vals = np.empty(out_ptr[-1])
    cols[pos], vals[pos] = t_idx, off
    cols[dpos], vals[dpos] = np.arange(n), diag
    keep = vals != 0.0
    rr = np.repeat(np.arange(n, dtype=np.int64), np.diff(out_ptr))[keep]
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rr, minlength=n), out=ptr[1:])
    return CSR(n, ptr, cols[keep], vals[keep])


def check_symmetric(m: CSR, rtol=1e-12):
    """sparse.py:100-105."""
    s = m.scipy()
    d = (s - s.T).tocsr()
    scale = float(np.max(np.abs(m.data))) if m.nnz else 0.0
    if d.nnz and np.max(np.abs(d.data)) > rtol * max(scale, 1.0):
        raise OracleInputError("matrix is not symmetric")


def identity_shift(q: CSR, seed=42):
    """operators.py:138-156."""
    check_symmetric(q)
    n = q.n
    if n == 0 or q.nnz == 0:
        return 0.0
    tau = 1e-8 * float(q.diagonal().sum()) / n
    if n <= DENSE_EPS_MAX_N:
        w = np.linalg.eigvalsh(q.dense())
        hit = w[w > tau]
        return float(hit[0]) if hit.size else 0.0
    return smallest_above_null(q, tau, seed=seed, tol=1e-6, max_iter=60)


def repulsion_weight(l: CSR, q: CSR, eps):
    """operators.py:159-176."""
    if l.n != q.n:
        raise OracleInputError("dimension mismatch")
    if eps < 0:
        raise OracleInputError("epsilon must be non-negative")
    dq = q.diagonal()
    denom = 2.0 * dq - q.row_sums()
    sel = dq > 0.0
    if not np.any(sel):
        return 0.0
    return float(np.min(eps / denom[sel]))


def assemble(l: CSR, q: CSR, mu, eps):
    """operators.py:179-186: ``(L - mu*Q) + eps*I`` with scipy's zero dropping.

    scipy's canonical CSR binop stores op(a, b) over the union pattern and
    drops exact zeros (F7); the two roundings (``L - mu*Q`` then ``+ eps``)
    are kept separate, exactly as the reference evaluates them.
    """
    if l.n != q.n:
        raise OracleInputError("dimension mismatch")
    import scipy.sparse as sp
    n = l.n
    step1 = l.scipy() - mu * q.scipy()
    m = step1 + eps * sp.identity(n, format="csr")
    m = sp.csr_matrix(m)
    m.sort_indices()
    return CSR(n, m.indptr, m.indices, m.data)


def gershgorin_radii(a: CSR):
    """sparse.py:84-94: off-diagonal |A_ij| summed sequentially per row."""
    r = a.rows()
    absd = np.abs(a.data)
    absd[r == a.indices] = 0.0
    return np.bincount(r, weights=absd, minlength=a.n)


def balance_radii(radii):
    """operators.py:189-202 (log-space, two mean passes)."""
    logr = np.log(np.asarray(radii, np.float64))
    logb = logr - logr.mean()
    logb -= logb.mean()
    return np.exp(logb), float(np.exp(logr.mean()))


def degree_balancing(a: CSR):
    """operators.py:205-219."""
    radii = gershgorin_radii(a)
    if np.any(radii <= 0.0):
        node = int(np.argmax(radii <= 0.0))
        raise OracleDisconnected(f"node {node} has no off-diagonal coupling; "
                                 "extract the largest connected component and retry")
    return balance_radii(radii)


def operator_pair(n, indptr, indices, weights, literal_diagonal=False, seed=42,
                  eps_override=None):
    """operators.py:222-233 chain.  Returns a dict of every intermediate."""
    l = laplacian(n, indptr, indices, weights)
    t_ptr, t_idx = two_hop(n, indptr, indices)
    q = q_matrix(n, t_ptr, t_idx, literal_diagonal)
    eps = identity_shift(q, seed) if eps_override is None else float(eps_override)
    mu = repulsion_weight(l, q, eps)
    a = assemble(l, q, mu, eps)
    b, gdeg = degree_balancing(a)
    return dict(L=l, t_ptr=t_ptr, t_idx=t_idx, Q=q, eps=eps, mu=mu, A=a, b=b,
                generalized_degree=gdeg)


def pair_diagnostics(a: CSR, q: CSR, mu, eps):
    """operators.py:76-85."""
    left = a.diagonal() - gershgorin_radii(a)
    binding = int(np.argmin(left))
    return {"mu": float(mu), "epsilon": float(eps),
            "min_disc_left_end": float(left[binding]), "q_nnz": int(q.nnz),
            "binding_row": binding}


# -- LOBPCG (eigensolver.py:92-283) ----------------------------------------------

def _b_project_out(y, block, b):
    """eigensolver.py:92-99."""
    by = b * y
    den = float(y @ by)
    if den <= 0.0:
        return block
    return block - np.outer(y, (block.T @ by) / den)


def _b_orthonormalize(blocks, ablocks, b, prefix=0):
    """eigensolver.py:102-153: bulk CGS2 against a trusted prefix, then
    column-wise CGS2 with the 1e-12 relative drop rule, mirrored on A-images."""
    S = np.concatenate(blocks, axis=1)
    AS = np.concatenate(ablocks, axis=1)
    n, s = S.shape
    Q = np.empty((n, s), order="F")
    AQ = np.empty((n, s), order="F")
    if prefix:
        Q[:, :prefix] = S[:, :prefix]
        AQ[:, :prefix] = AS[:, :prefix]
        V = np.asfortranarray(S[:, prefix:])
        AV = np.asfortranarray(AS[:, prefix:])
        lead, alead = Q[:, :prefix], AQ[:, :prefix]
        for _ in range(2):
            c = lead.T @ (b[:, None] * V)
            V -= lead @ c
            AV -= alead @ c
    else:
        V = np.asfortranarray(S)
        AV = np.asfortranarray(AS)
    kept = prefix
    biggest = 1.0 if prefix else 0.0
    for j in range(s - prefix):
        v, av = V[:, j], AV[:, j]
        for _ in range(2):
            if kept > prefix:
                basis = Q[:, prefix:kept]
                c = basis.T @ (b * v)
                v -= basis @ c
                av -= AQ[:, prefix:kept] @ c
        nrm = float(np.sqrt(max(v @ (b * v), 0.0)))
        biggest = max(biggest, nrm)
        if nrm == 0.0 or nrm < DROP_REL * biggest:
            continue
        Q[:, kept] = v / nrm
        AQ[:, kept] = av / nrm
        kept += 1
    return Q[:, :kept], AQ[:, :kept]


def initial_block(n, k, seed):
    """eigensolver.py:177-178: PCG64(seed).standard_normal((n, k)), plus the
    generator so refills continue the same stream (eigensolver.py:189)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, k)), rng


def _signs(vecs):
    """eigensolver.py:83-89: largest |entry| positive, first index on ties."""
    for j in range(vecs.shape[1]):
        lead = int(np.argmax(np.abs(vecs[:, j])))
        if vecs[lead, j] < 0.0:
            vecs[:, j] = -vecs[:, j]
    return vecs


def lobpcg(a: CSR, b, k, tol=1e-8, max_iter=500, seed=42, preconditioner="jacobi",
           deflate=None, x0=None, iter_times=None):
    """eigensolver.py:156-283.  Returns a dict with the EigenResult fields.
    ``iter_times`` (a list, optional) receives the wall time of every
    iteration of the main loop (bench.py's CPU baseline)."""
    import time as _time
    n = a.n
    b = np.asarray(b, np.float64)
    if b.shape != (n,):
        raise OracleInputError("diagonal length does not match n")
    if np.any(b <= 0.0) or not np.all(np.isfinite(b)):
        raise OracleInputError("diagonal entries must be strictly positive and finite")
    if k > n:
        raise OracleInputError(f"block size {k} exceeds dimension {n}")
    X, rng = initial_block(n, k, seed)
    if x0 is not None:
        X = np.array(x0, dtype=np.float64, copy=True)
    defl = None
    if deflate is not None:
        defl = np.atleast_2d(np.asarray(deflate, np.float64).T).T
        for y in defl.T:
            X = _b_project_out(y, X, b)

    def orth_refill(blocks, ablocks):
        S, AS = _b_orthonormalize(blocks, ablocks, b)
        while S.shape[1] < k:
            extra = rng.standard_normal((n, k - S.shape[1]))
            if defl is not None:
                for y in defl.T:
                    extra = _b_project_out(y, extra, b)
            S, AS = _b_orthonormalize([S, extra], [AS, a.matmat(extra)], b)
        return S, AS

    def ritz(Xb, AXb):
        g = Xb.T @ AXb
        th, Y = np.linalg.eigh(0.5 * (g + g.T))
        return th[:k], Y[:, :k]

    X, AX = orth_refill([X], [a.matmat(X)])
    theta, Y = ritz(X, AX)
    X, AX = X @ Y, AX @ Y

    anorm = a.frobenius() / np.sqrt(n)
    bmax = float(b.max())
    if preconditioner == "jacobi":
        d = a.diagonal().copy()
        d[d <= 0.0] = 1.0
        prec = 1.0 / d
    else:
        prec = None

    def resid(Xb, AXb, th):
        R = AXb - (b[:, None] * Xb) * th
        rn = np.linalg.norm(R, axis=0)
        qn = np.linalg.norm(Xb, axis=0)
        return R, rn, rn <= tol * ((anorm + np.abs(th) * bmax) * qn)

    P = AP = None
    history = []
    it = 0
    for it in range(1, max_iter + 1):
        t_it = _time.perf_counter()
        R, rn, conv = resid(X, AX, theta)
        history.append(float(theta.sum()))
        if conv.all():
            AX = a.matmat(X)
            g = X.T @ AX
            theta = np.diag(0.5 * (g + g.T)).copy()
            R, rn, conv = resid(X, AX, theta)
            if conv.all():
                break
        W = R[:, ~conv]
        if prec is not None:
            W = prec[:, None] * W
        if defl is not None:
            for y in defl.T:
                W = _b_project_out(y, W, b)
        blocks, ablocks = [X, W], [AX, a.matmat(W)]
        if P is not None and P.shape[1]:
            blocks.append(P)
            ablocks.append(AP)
        S, AS = _b_orthonormalize(blocks, ablocks, b,
                                  prefix=X.shape[1] if it % 32 else 0)
        g = S.T @ AS
        th_all, Y = np.linalg.eigh(0.5 * (g + g.T))
        take = min(k, S.shape[1])
        theta, Y = th_all[:take], Y[:, :take]
        X, AX = S @ Y, AS @ Y
        P, AP = S[:, k:] @ Y[k:, :], AS[:, k:] @ Y[k:, :]
        if take < k:
            X, AX = orth_refill([X], [AX])
            theta, Y = ritz(X, AX)
            X, AX = X @ Y, AX @ Y
            P = AP = None
        if iter_times is not None:
            iter_times.append(_time.perf_counter() - t_it)

    AX = a.matmat(X)
    g = X.T @ AX
    theta = np.diag(0.5 * (g + g.T)).copy()
    order = np.argsort(theta, kind="stable")
    theta, X, AX = theta[order], X[:, order], AX[:, order]
    _, rn, conv = resid(X, AX, theta)
    X = _signs(X)
    return dict(eigenvalues=theta, eigenvectors=X, iterations=it,
                residual_norms=rn, converged=conv, ritz_sum_history=history)


def smallest_above_null(m: CSR, tau, seed=42, tol=1e-8, max_iter=500):
    """eigensolver.py:431-460."""
    n = m.n
    if n <= DENSE_EPS_MAX_N:
        w = np.linalg.eigvalsh(m.dense())
        hit = w[w > tau]
        return float(hit[0]) if hit.size else 0.0
    const = np.full(n, 1.0 / np.sqrt(n))
    k = 8
    while True:
        res = lobpcg(m, np.ones(n), min(k, n - 1), tol=tol, max_iter=max_iter,
                     seed=seed, deflate=const)
        ev = res["eigenvalues"]
        hit = ev[ev > tau]
        if hit.size:
            return float(hit[0])
        if k >= min(64, n - 1):
            return 0.0
        k *= 2


def _solve_drop_first(a, b, k, tol, max_iter, seed, preconditioner, require):
    """embedding.py:61-74 + eigensolver.py:471-481."""
    res = lobpcg(a, b, k + 1, tol=tol, max_iter=max_iter, seed=seed,
                 preconditioner=preconditioner)
    if require and not res["converged"].all():
        bad = int(np.sum(~res["converged"]))
        raise OracleConvergence(f"{bad} of {res['converged'].size} eigenpairs "
                                f"unconverged after {res['iterations']} iterations", res)
    return res


def embed(n, indptr, indices, weights, k, tol=1e-8, max_iter=500, seed=42,
          preconditioner="jacobi", literal_diagonal=False, require_convergence=True,
          check_connected=True):
    """embedding.py:77-103 (``check_connected=False`` bypasses
    ``_check_embeddable``'s component test, as SURVEY F6 does for config 4)."""
    if not 1 <= k <= n - 1:
        raise OracleInputError("embedding dimension out of range")
    if check_connected:
        count, _ = components(n, indptr, indices)
        if count != 1:
            raise OracleDisconnected(f"graph has {count} connected components", count)
    pair = operator_pair(n, indptr, indices, weights, literal_diagonal, seed)
    res = _solve_drop_first(pair["A"], pair["b"], k, tol, max_iter, seed,
                            preconditioner, require_convergence)
    diag = pair_diagnostics(pair["A"], pair["Q"], pair["mu"], pair["eps"])
    diag.update({"iterations": int(res["iterations"]),
                 "residuals": [float(r) for r in res["residual_norms"]],
                 "converged": [bool(c) for c in res["converged"]],
                 "dropped_eigenvalue": float(res["eigenvalues"][0])})
    return dict(P=res["eigenvectors"][:, 1:], eigenvalues=res["eigenvalues"][1:],
                b=pair["b"], diagnostics=diag, pair=pair, result=res)


def laplacian_eigenmaps(n, indptr, indices, weights, k, tol=1e-8, max_iter=500,
                        seed=42, preconditioner="jacobi", require_convergence=True):
    """embedding.py:106-127."""
    if not 1 <= k <= n - 1:
        raise OracleInputError("embedding dimension out of range")
    count, _ = components(n, indptr, indices)
    if count != 1:
        raise OracleDisconnected(f"graph has {count} connected components", count)
    l = laplacian(n, indptr, indices, weights)
    res = _solve_drop_first(l, np.ones(n), k, tol, max_iter, seed, preconditioner,
                            require_convergence)
    return dict(P=res["eigenvectors"][:, 1:], eigenvalues=res["eigenvalues"][1:],
                result=res)


def dense_generalized_eigh(a: CSR, b, k):
    """Dense check: eigh(B^-1/2 A B^-1/2), vectors mapped back
    with B^-1/2 and sign-fixed like eigensolver.py:83-89.  Stands in for the
    reference's cyclic-Jacobi ``dense_oracle`` (eigensolver.py:396-425)."""
    b = np.asarray(b, np.float64)
    s = 1.0 / np.sqrt(b)
    c = a.dense() * s[:, None] * s[None, :]
    w, v = np.linalg.eigh(0.5 * (c + c.T))
    return w[:k], _signs(s[:, None] * v[:, :k])


# ------------------------------------------------------------ clustering ---
# C4 readout: rng.py:9-127 and clustering.py:50-134.
_M64 = (1 << 64) - 1


def _mix64(x):
    """rng.py:49-54 (splitmix64 finalizer)."""
    x &= _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return (x ^ (x >> 31)) & _M64


def stream_seed(seed, index):
    """rng.py:65-67."""
    return _mix64((_mix64(seed) + ((index + 1) * 0xD2B74407B1CE6E93 & _M64)) & _M64)


class Xoshiro256:
    """rng.py:74-127 (xoshiro256** seeded by four splitmix64 outputs)."""

    def __init__(self, seed):
        z, s = seed & _M64, []
        for _ in range(4):
            z = (z + 0x9E3779B97F4A7C15) & _M64
            s.append(_mix64(z))
        if not any(s):
            s[0] = 1
        self.s = s

    def next_u64(self):
        s0, s1, s2, s3 = self.s
        rot = lambda x, r: ((x << r) | (x >> (64 - r))) & _M64  # noqa: E731
        out = (rot((s1 * 5) & _M64, 7) * 9) & _M64
        t = (s1 << 17) & _M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        self.s = [s0, s1, s2, rot(s3, 45)]
        return out

    def uniform(self):
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def index(self, n):
        i = int(self.uniform() * n)
        return n - 1 if i >= n else i

    def weighted_index(self, cum):
        total = float(cum[-1])
        if total <= 0.0:
            return self.index(len(cum))
        return int(np.searchsorted(cum, self.uniform() * total, side="right"))


def normalize_rows(pts):
    """clustering.py:50-56."""
    pts = np.asarray(pts, np.float64)
    nr = np.linalg.norm(pts, axis=1, keepdims=True)
    return np.where(nr > 0.0, pts / np.where(nr > 0.0, nr, 1.0), pts)


def kmeans(pts, c, restarts=20, seed=42):
    """clustering.py:99-134 (k-means++ :57-67, Lloyd :70-96); returns (labels, wcss)."""
    pts = np.asarray(pts, np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    n = pts.shape[0]
    if not 1 <= c <= n or restarts < 1:
        raise OracleInputError("bad cluster count / restarts")
    if c == 1:
        return np.zeros(n, np.int64), 0.0
    if c == n:
        return np.arange(n, dtype=np.int64), 0.0
    best = None
    for r in range(restarts):
        rng = Xoshiro256(stream_seed(seed, r))
        centers = np.empty((c, pts.shape[1]))
        centers[0] = pts[rng.index(n)]
        d2 = np.sum((pts - centers[0]) ** 2, axis=1)
        for j in range(1, c):
            centers[j] = pts[rng.weighted_index(np.cumsum(d2))]
            d2 = np.minimum(d2, np.sum((pts - centers[j]) ** 2, axis=1))
        labels = np.full(n, -1, dtype=np.int64)
        for _ in range(300):
            dd = (np.sum(pts * pts, axis=1)[:, None] - 2.0 * (pts @ centers.T)
                  + np.sum(centers * centers, axis=1)[None, :])
            new = np.argmin(dd, axis=1)
            for j in range(c):
                if not np.any(new == j):
                    fit = dd[np.arange(n), new]
                    fit = np.where(np.bincount(new, minlength=c)[new] > 1, fit, -np.inf)
                    new[int(np.argmax(fit))] = j
            if np.array_equal(new, labels):
                break
            labels = new
            for j in range(c):
                mem = pts[labels == j]
                if mem.size:
                    centers[j] = mem.mean(axis=0)
        wcss = float(np.sum((pts - centers[labels]) ** 2))
        if best is None or wcss < best[1]:
            best = (labels, wcss)
    return best


def knn_graph(X, k, weighted=True):
    """graph.py:281-315 (dense distances, stable argsort, union, mean-d2 bandwidth)
    -> canonical CSR (graph.py:31-79); returns (n, indptr, indices, weights)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise OracleInputError("feature matrix must be 2-D")
    n = X.shape[0]
    if not 1 <= k < n:
        raise OracleInputError(f"k must satisfy 1 <= k < n, got k={k}, n={n}")
    sq = np.sum(X * X, axis=1)
    d2 = sq[:, None] + sq[None, :] - 2.0 * (X @ X.T)
    np.maximum(d2, 0.0, out=d2)
    np.fill_diagonal(d2, np.inf)
    nearest = np.argsort(d2, axis=1, kind="stable")[:, :k]
    i = np.repeat(np.arange(n), k)
    j = nearest.ravel()
    key = np.unique(np.minimum(i, j) * n + np.maximum(i, j))
    ii, jj = key // n, key % n
    if weighted:
        dist2 = d2[ii, jj]
        sigma2 = float(dist2.mean())
        w = np.exp(-dist2 / sigma2) if sigma2 > 0.0 else np.ones_like(dist2)
    else:
        w = np.ones(key.size)
    bad = ~((w > 0.0) & np.isfinite(w))
    if np.any(bad):
        e = int(np.argmax(bad))
        raise OracleInputError(f"edge ({ii[e]}, {jj[e]}) has non-positive weight {w[e]}")
    src = np.concatenate([ii, jj])
    dst = np.concatenate([jj, ii])
    wts = np.concatenate([w, w])
    order = np.lexsort((dst, src))
    indptr = np.zeros(n + 1, np.int64)
    np.add.at(indptr, src[order] + 1, 1)
    np.cumsum(indptr, out=indptr)
    return n, indptr, dst[order], wts[order]
