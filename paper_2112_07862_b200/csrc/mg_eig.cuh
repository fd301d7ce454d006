// Smallest eigenpairs of a small dense symmetric matrix by ONE thread block:
// the device replacement of np.linalg.eigh in the Rayleigh-Ritz step
// (eigensolver.py:198, 252, 263), which only ever uses the `take` smallest
// pairs.  Householder tridiagonalisation, multisection (parallel Sturm
// counts) for the wanted eigenvalues, inverse iteration for the vectors,
// Gram-Schmidt (cluster safety), Householder back-transformation.
// Accuracy is absolute ~eps*||A||, like LAPACK syevd.  All dot products are
// warp-cooperative; block reductions use shuffles + one shared-memory stage.
#pragma once
#include <float.h>

#include "mg_common.cuh"

namespace mg {

static constexpr int kEigMaxN = 256;

struct EigWork {
  double *tau;   // n
  double *d;     // n
  double *e;     // n (e[i] couples i, i+1)
  double *lo;    // nev
  double *hi;    // nev
  int *cnt;      // nev * P  (P <= blockDim / nev)
  double *red;   // blockDim (p vector of the Householder step, coefficients)
  double *red2;  // >= 32 (warp partials)
  double *lu;    // unused (kept for ABI of callers)
  long long *clk = nullptr;  // optional section timestamps (thread 0), 6 entries
};

// block-wide sum; every thread gets the result.  `wp` needs 32 doubles.
__device__ __forceinline__ double blk_sum(double v, double *wp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) wp[warp] = v;
  __syncthreads();
  double t = lane < nw ? wp[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

__device__ __forceinline__ int sturm_count(const double *d, const double *e, int n, double x,
                                           double pivmin) {
  double q = d[0] - x;
  int c = q < 0.0 ? 1 : 0;
  for (int i = 1; i < n; ++i) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
    c += q < 0.0 ? 1 : 0;
  }
  return c;
}

// A: n x n symmetric (lda), destroyed (Householder vectors stored below the
// diagonal).  On exit w[0..nev) ascending and Z[i * ldz + j] (n x nev) the
// matching orthonormal eigenvectors.  n <= kEigMaxN, blockDim multiple of 32.
__device__ inline void blk_eig_smallest(double *A, int lda, int n, int nev, double *w, double *Z,
                                        int ldz, EigWork wk) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double *tau = wk.tau, *d = wk.d, *e = wk.e, *p = wk.red, *wp = wk.red2;
  if (wk.clk && tid == 0) wk.clk[0] = clock64();
  // ---- 1. Householder reduction to tridiagonal form (lower) ----
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    double *x = A + (k + 1) * lda + k;  // column below the diagonal: x[i*lda], i < m
    double s = 0.0;
    for (int i = 1 + tid; i < m; i += nt) s += x[i * lda] * x[i * lda];
    const double sigma = blk_sum(s, wp);
    const double x0 = x[0];
    if (sigma == 0.0) {
      __syncthreads();
      if (tid == 0) {
        tau[k] = 0.0;
        e[k] = x0;
      }
      continue;
    }
    const double nrm = sqrt(x0 * x0 + sigma);
    const double alpha = x0 <= 0.0 ? nrm : -nrm;
    const double v0 = x0 - alpha;
    const double tk = 2.0 / (v0 * v0 + sigma);
    __syncthreads();
    if (tid == 0) {
      x[0] = v0;
      tau[k] = tk;
      e[k] = alpha;
    }
    __syncthreads();
    // p = tau * A22 v : 4 lanes per row
    const double *A22 = A + (k + 1) * lda + (k + 1);
    const int rows_per_pass = nt >> 2;
    const int passes = (m + rows_per_pass - 1) / rows_per_pass;  // uniform trip count
    for (int ps = 0; ps < passes; ++ps) {
      const int base = ps * rows_per_pass + (tid >> 2);
      double acc = 0.0;
      if (base < m) {
        const double *row = A22 + base * lda;
        for (int c = tid & 3; c < m; c += 4) acc += row[c] * x[c * lda];
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (base < m && (tid & 3) == 0) p[base] = tk * acc;
    }
    __syncthreads();
    double s2 = 0.0;
    for (int i = tid; i < m; i += nt) s2 += x[i * lda] * p[i];
    const double K = 0.5 * tk * blk_sum(s2, wp);
    for (int i = tid; i < m; i += nt) p[i] -= K * x[i * lda];
    __syncthreads();
    // rank-2 update, one warp per row (no per-element integer division)
    double *A22w = A + (k + 1) * lda + (k + 1);
    for (int r = warp; r < m; r += nw) {
      const double xr = x[r * lda], pr = p[r];
      double *row = A22w + r * lda;
      for (int c = lane; c < m; c += 32) row[c] -= xr * p[c] + pr * x[c * lda];
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += nt) d[i] = A[i * lda + i];
  if (tid == 0 && n >= 2) {
    e[n - 2] = A[(n - 1) * lda + (n - 2)];
    tau[n - 2] = 0.0;
  }
  __syncthreads();
  if (wk.clk && tid == 0) wk.clk[1] = clock64();
  // ---- 2. multisection for eigenvalues 0..nev-1 ----
  double gl = INFINITY, gu = -INFINITY, emax = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - r);
    gu = fmax(gu, d[i] + r);
    emax = fmax(emax, fabs(d[i]) + r);
  }
  const double scale = fmax(emax, DBL_MIN);
  gl -= 4.0 * DBL_EPSILON * scale + DBL_MIN;
  gu += 4.0 * DBL_EPSILON * scale + DBL_MIN;
  const double pivmin = DBL_MIN * fmax(1.0, emax * emax);
  const int P = max(1, min(63, nt / max(nev, 1) - 1));
  for (int j = tid; j < nev; j += nt) {
    wk.lo[j] = gl;
    wk.hi[j] = gu;
  }
  __syncthreads();
  for (int iter = 0; iter < 80; ++iter) {
    for (int t = tid; t < nev * P; t += nt) {
      const int j = t / P, q = t - j * P;
      const double l = wk.lo[j], h = wk.hi[j];
      wk.cnt[t] = sturm_count(d, e, n, l + (h - l) * (double)(q + 1) / (double)(P + 1), pivmin);
    }
    __syncthreads();
    double open = 0.0;
    for (int j = tid; j < nev; j += nt) {
      const double l = wk.lo[j], h = wk.hi[j];
      if (h - l <= 2.0 * DBL_EPSILON * fmax(fabs(l), fabs(h)) + 2.0 * pivmin) continue;
      int q = 0;
      while (q < P && wk.cnt[j * P + q] <= j) ++q;
      const double nl = q == 0 ? l : l + (h - l) * (double)q / (double)(P + 1);
      const double nh = q == P ? h : l + (h - l) * (double)(q + 1) / (double)(P + 1);
      wk.lo[j] = nl;
      wk.hi[j] = nh;
      if (nh - nl > 2.0 * DBL_EPSILON * fmax(fabs(nl), fabs(nh)) + 2.0 * pivmin) open += 1.0;
    }
    if (blk_sum(open, wp) == 0.0) break;
  }
  __syncthreads();
  for (int j = tid; j < nev; j += nt) w[j] = 0.5 * (wk.lo[j] + wk.hi[j]);
  __syncthreads();
  if (wk.clk && tid == 0) wk.clk[2] = clock64();
  // ---- 3. inverse iteration, one thread per eigenvector (LU in local memory) ----
  for (int j = tid; j < nev; j += nt) {
    double ua[kEigMaxN], ub[kEigMaxN], uc[kEigMaxN], lm[kEigMaxN];
    unsigned char sw[kEigMaxN];
    const double lam = w[j];
    const double tiny = DBL_EPSILON * scale + pivmin;
    for (int i = 0; i < n; ++i) {
      ua[i] = d[i] - lam;
      ub[i] = i + 1 < n ? e[i] : 0.0;
      uc[i] = 0.0;
    }
    for (int i = 0; i + 1 < n; ++i) {
      const double sub = e[i];  // original (i+1, i) entry
      if (fabs(ua[i]) >= fabs(sub)) {
        sw[i] = 0;
        const double piv = ua[i] != 0.0 ? ua[i] : tiny;
        ua[i] = piv;
        const double l = sub / piv;
        lm[i] = l;
        ua[i + 1] -= l * ub[i];
      } else {
        sw[i] = 1;
        const double l = ua[i] / sub;
        lm[i] = l;
        const double ai1 = ua[i + 1], bi1 = ub[i + 1], bi = ub[i];
        ua[i] = sub;
        ub[i] = ai1;
        uc[i] = bi1;
        ua[i + 1] = bi - l * ai1;
        ub[i + 1] = -l * bi1;
      }
    }
    if (ua[n - 1] == 0.0) ua[n - 1] = tiny;
    double *z = Z + j;
    uint32_t h = 2654435761u * (uint32_t)(j + 1) + 12345u;
    for (int i = 0; i < n; ++i) {
      h ^= h << 13;
      h ^= h >> 17;
      h ^= h << 5;
      z[i * ldz] = (double)(h & 0xffff) / 65535.0 - 0.5 + 1e-3;
    }
    for (int sweep = 0; sweep < 2; ++sweep) {
      for (int i = 0; i + 1 < n; ++i) {
        if (sw[i]) {
          const double t = z[i * ldz];
          z[i * ldz] = z[(i + 1) * ldz];
          z[(i + 1) * ldz] = t - lm[i] * z[i * ldz];
        } else {
          z[(i + 1) * ldz] -= lm[i] * z[i * ldz];
        }
      }
      double nrm = 0.0;
      for (int i = n - 1; i >= 0; --i) {
        double s = z[i * ldz];
        if (i + 1 < n) s -= ub[i] * z[(i + 1) * ldz];
        if (i + 2 < n) s -= uc[i] * z[(i + 2) * ldz];
        s /= ua[i];
        z[i * ldz] = s;
        nrm += s * s;
      }
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = 0; i < n; ++i) z[i * ldz] *= inv;
    }
  }
  __syncthreads();
  if (wk.clk && tid == 0) wk.clk[3] = clock64();
  // ---- 4. Gram-Schmidt (CGS2) in eigenvalue order; one warp per coefficient ----
  for (int j = 1; j < nev; ++j) {
    for (int rep = 0; rep < 2; ++rep) {
      for (int i = warp; i < j; i += nw) {
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s += Z[r * ldz + i] * Z[r * ldz + j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) p[i] = s;
      }
      __syncthreads();
      for (int r = tid; r < n; r += nt) {
        double s = 0.0;
        for (int i = 0; i < j; ++i) s += p[i] * Z[r * ldz + i];
        Z[r * ldz + j] -= s;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int r = tid; r < n; r += nt) s += Z[r * ldz + j] * Z[r * ldz + j];
    const double ss = blk_sum(s, wp);
    const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
    for (int r = tid; r < n; r += nt) Z[r * ldz + j] *= inv;
    __syncthreads();
  }
  if (wk.clk && tid == 0) wk.clk[4] = clock64();
  // ---- 5. back-transformation Z <- H_0 ... H_{n-3} Z ; one warp per column dot ----
  for (int k = n - 3; k >= 0; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    const int m = n - k - 1;
    const double *v = A + (k + 1) * lda + k;
    for (int j = warp; j < nev; j += nw) {
      double s = 0.0;
      for (int i = lane; i < m; i += 32) s += v[i * lda] * Z[(k + 1 + i) * ldz + j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) p[j] = tk * s;
    }
    __syncthreads();
    for (int i = warp; i < m; i += nw) {
      const double vi = v[i * lda];
      double *zr = Z + (k + 1 + i) * ldz;
      for (int j = lane; j < nev; j += 32) zr[j] -= vi * p[j];
    }
    __syncthreads();
  }
  if (wk.clk && tid == 0) wk.clk[5] = clock64();
}

}  // namespace mg
