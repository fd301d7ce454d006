// Small dense linear algebra executed by ONE thread block (device side of the
// Rayleigh-Ritz step and of the B-orthonormalisation).  Replaces the LAPACK
// calls of the reference (np.linalg.eigh at eigensolver.py:198, 252, 263;
// eigvalsh at operators.py:151) and the column-sweep norm/drop logic of
// _b_mgs_pair (eigensolver.py:102-153) expressed as a Cholesky factorisation
// of the B-Gram matrix.  All routines are called by every thread of the block.
#pragma once
#include <float.h>

#include "mg_common.cuh"

namespace mg {

// Right-looking Cholesky with the reference's drop rule: column a (in the
// given order) is dropped when its post-projection B-norm -- the pivot --
// is 0 or below 1e-12 * (largest pivot seen so far, starting at maxnorm0).
// G (nl x nl, ld) is overwritten; on exit R holds the upper factor over the
// logical index space (rows/cols of dropped columns are zero), keep[a] = 1
// for kept columns.  Returns the kept count (same value in every thread).
//
// Gram-based factorisation cannot resolve a column whose post-projection norm
// is below ~sqrt(eps) of its own norm (the pivot is a cancellation of two
// nearly equal Gram quantities), so such columns are also dropped: rel_tol
// bounds pivot / sqrt(G_aa(original)).  This is the only deliberate
// deviation from the reference's column-sweep MGS, which can keep them; the
// dropped direction carries < rel_tol of its column.
__device__ inline int blk_cholesky_drop(double *G, int ld, int nl, double maxnorm0, double *R,
                                        int ldr, int *keep, double *orig, double rel_tol,
                                        double abs_tol = 1e-12) {
  int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < nl * nl; e += nt) R[(e / nl) * ldr + (e % nl)] = 0.0;
  for (int a = tid; a < nl; a += nt) orig[a] = G[a * ld + a];
  double maxnorm = maxnorm0;
  int kept = 0;
  __syncthreads();
  for (int a = 0; a < nl; ++a) {
    double d = G[a * ld + a];
    double nrm = sqrt(d > 0.0 ? d : 0.0);
    maxnorm = fmax(maxnorm, nrm);
    double o = orig[a];
    bool drop = (nrm == 0.0) || (nrm < abs_tol * maxnorm) ||
                (nrm < rel_tol * sqrt(o > 0.0 ? o : 0.0));
    if (tid == 0) keep[a] = drop ? 0 : 1;
    if (drop) continue;  // uniform across threads (all read the same G entry)
    ++kept;
    double inv = 1.0 / nrm;
    for (int b = a + tid; b < nl; b += nt) R[a * ldr + b] = (b == a) ? nrm : G[a * ld + b] * inv;
    __syncthreads();
    int rem = nl - a - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      int b = a + 1 + e / rem, c = a + 1 + e % rem;
      G[b * ld + c] -= R[a * ldr + b] * R[a * ldr + c];
    }
    __syncthreads();
  }
  __syncthreads();
  return kept;
}

// Inverse of the upper-triangular factor restricted to kept columns.
// R (nl x nl over logical indices, zero rows/cols for dropped) -> Rinv with
// the same index space: V1[:, t] = sum_a V[:, a] * Rinv[a][t] for kept t.
__device__ inline void blk_tri_inv_kept(const double *R, int ldr, int nl, const int *keep,
                                        double *Rinv, int ldi) {
  int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < nl * nl; e += nt) Rinv[(e / nl) * ldi + (e % nl)] = 0.0;
  __syncthreads();
  for (int t = tid; t < nl; t += nt) {
    if (!keep[t]) continue;
    Rinv[t * ldi + t] = 1.0 / R[t * ldr + t];
    for (int u = t - 1; u >= 0; --u) {
      if (!keep[u]) continue;
      double s = 0.0;
      for (int v = u + 1; v <= t; ++v)
        if (keep[v]) s += R[u * ldr + v] * Rinv[v * ldi + t];
      Rinv[u * ldi + t] = -s / R[u * ldr + u];
    }
  }
  __syncthreads();
}

// Parallel cyclic Jacobi (round-robin pair ordering) on a symmetric n x n
// matrix A (ld lda), accumulating rotations into V (ld ldv, may be null).
// On exit the eigenvalues are in w[0..n) ascending and the columns of V are
// permuted accordingly (stable in the original column index).
// Scratch: cs (2 * (n/2+1) doubles), perm (n ints), cnt (1 int), all shared.
__device__ inline void blk_jacobi(double *A, int lda, int n, double *V, int ldv, double *w,
                                  double *cs, int *pidx, int *perm, int *cnt, double *red) {
  int tid = threadIdx.x, nt = blockDim.x;
  if (V)
    for (int e = tid; e < n * n; e += nt) V[(e / n) * ldv + (e % n)] = (e / n == e % n) ? 1.0 : 0.0;
  // Frobenius norm
  double s = 0.0;
  for (int e = tid; e < n * n; e += nt) {
    double x = A[(e / n) * lda + (e % n)];
    s += x * x;
  }
  red[tid] = s;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  double fro = sqrt(red[0]);
  __syncthreads();
  // rotate only couplings that can still move an eigenvalue by more than
  // ~eps*||A||_F (absolute accuracy, like LAPACK syevd); relative criterion
  // below it would force extra sweeps for the tiny Ritz values
  double abs_floor = 0.25 * DBL_EPSILON * fro;
  int np = (n + 1) & ~1;  // even player count; player n (if odd) is a bye
  int half = np / 2;
  for (int sweep = 0; sweep < 60 && n > 1; ++sweep) {
    if (tid == 0) *cnt = 0;
    __syncthreads();
    for (int r = 0; r < np - 1; ++r) {
      // pairs of round r (circle method): (np-1, r) and ((r+k)%(np-1), (r-k+np-1)%(np-1))
      for (int k = tid; k < half; k += nt) {
        int p, q;
        if (k == 0) {
          p = np - 1;
          q = r;
        } else {
          p = (r + k) % (np - 1);
          q = (r - k + np - 1) % (np - 1);
        }
        if (p > q) { int t = p; p = q; q = t; }
        double c = 1.0, sn = 0.0;
        if (q < n) {
          double apq = A[p * lda + q];
          double app = A[p * lda + p], aqq = A[q * lda + q];
          if (apq != 0.0 && fabs(apq) > abs_floor &&
              fabs(apq) > DBL_EPSILON * sqrt(fabs(app) * fabs(aqq))) {
            double th = (aqq - app) / (2.0 * apq);
            double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
            atomicAdd(cnt, 1);
          }
        }
        pidx[2 * k] = p;
        pidx[2 * k + 1] = q;
        cs[2 * k] = c;
        cs[2 * k + 1] = sn;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = tid; e < half * n; e += nt) {
        int k = e / n, j = e % n;
        int p = pidx[2 * k], q = pidx[2 * k + 1];
        double sn = cs[2 * k + 1];
        if (q >= n || sn == 0.0) continue;
        double c = cs[2 * k];
        double ap = A[p * lda + j], aq = A[q * lda + j];
        A[p * lda + j] = c * ap - sn * aq;
        A[q * lda + j] = sn * ap + c * aq;
      }
      __syncthreads();
      // cols: A <- A J ; V <- V J
      for (int e = tid; e < half * n; e += nt) {
        int k = e / n, i = e % n;
        int p = pidx[2 * k], q = pidx[2 * k + 1];
        double sn = cs[2 * k + 1];
        if (q >= n || sn == 0.0) continue;
        double c = cs[2 * k];
        double ap = A[i * lda + p], aq = A[i * lda + q];
        A[i * lda + p] = c * ap - sn * aq;
        A[i * lda + q] = sn * ap + c * aq;
        if (V) {
          double vp = V[i * ldv + p], vq = V[i * ldv + q];
          V[i * ldv + p] = c * vp - sn * vq;
          V[i * ldv + q] = sn * vp + c * vq;
        }
      }
      __syncthreads();
      for (int k = tid; k < half; k += nt) {
        int p = pidx[2 * k], q = pidx[2 * k + 1];
        if (q < n && cs[2 * k + 1] != 0.0) {
          A[p * lda + q] = 0.0;
          A[q * lda + p] = 0.0;
        }
      }
      __syncthreads();
    }
    int c = *cnt;
    __syncthreads();
    if (c == 0) break;
  }
  // sort eigenvalues ascending (stable); NaN sorts last so perm is always a
  // permutation (the caller flags non-finite input separately)
  for (int i = tid; i < n; i += nt) {
    double di = A[i * lda + i];
    bool ni = di != di;
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      double dj = A[j * lda + j];
      bool nj = dj != dj;
      bool before = ni ? (nj && j < i) : (nj ? false : (dj < di || (dj == di && j < i)));
      if (!ni && nj) before = false;
      if (ni && !nj) before = true;
      if (before) ++rank;
    }
    perm[rank] = i;
  }
  __syncthreads();
  for (int i = tid; i < n; i += nt) w[i] = A[perm[i] * lda + perm[i]];
  __syncthreads();
}

// flag (atomicOr into *flag) if any of the n x n entries is not finite
__device__ inline void blk_check_finite(const double *A, int lda, int rows, int cols, int *flag,
                                        int bit) {
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    double v = A[(e / cols) * lda + (e % cols)];
    if (!isfinite(v)) atomicOr(flag, bit);
  }
}

}  // namespace mg
