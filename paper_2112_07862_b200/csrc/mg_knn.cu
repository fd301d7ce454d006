// Symmetrized k-nearest-neighbour graph (graph.py:281-315 of the reference,
// SURVEY 8(f).2) on the device: exact brute force over all pairs, the same
// distance arithmetic as the reference's dense matrix, the same union /
// bandwidth / weight rules and the same canonical CSR (Graph.from_edges).
//
// Reference arithmetic, restated:
//   sq_i   = sum_q x_iq^2                          (numpy row sum, sequential)
//   d2_ij  = max((sq_i + sq_j) - 2 (X X^T)_ij, 0), d2_ii = inf
//            (X X^T from BLAS syrk: a fused multiply-add chain over q -- this
//            matches OpenBLAS bit for bit off the diagonal for d <= 5, checked
//            in tests/test_knn.py; larger d can differ in the last bit)
//   row i keeps its k smallest d2 (stable argsort: ties -> lower index)
//   pairs  = union of {min(i,j), max(i,j)}, sorted
//   sigma2 = mean(d2 over pairs) (numpy pairwise summation, restated exactly)
//   w      = exp(-d2 / sigma2)  (exp within 1 ulp of numpy's), or 1
//   from_edges: every w must be finite and > 0, CSR of both half-edges sorted
//            by (row, column).
// Cost O(n^2 d) like the reference (which is O(n^2) in memory as well); the
// configs' large graphs come from synthetic.py's tree-based harness instead.
#include <cub/cub.cuh>
#include <vector>

#include "mg_common.cuh"
#include "mg_knn.cuh"

namespace mg {

namespace {

constexpr int kKnnThreads = 128;
constexpr int kKnnTileDoubles = 5120;  // 40 KB candidate tile
constexpr int kKnnMaxK = 64;

__global__ void k_knn_sq(int64_t n, int d, const double *__restrict__ X, double *__restrict__ sq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < d; ++q) s = __dadd_rn(s, __dmul_rn(X[i * d + q], X[i * d + q]));
    sq[i] = s;
  }
}

__device__ __forceinline__ double pair_d2(const double *xi, const double *xj, int d, double sqi,
                                          double sqj) {
  double dot = 0.0;
  for (int q = 0; q < d; ++q) dot = fma(xi[q], xj[q], dot);
  const double v = __dsub_rn(__dadd_rn(sqi, sqj), __dmul_rn(2.0, dot));
  return v > 0.0 ? v : 0.0;  // np.maximum(d2, 0.0) (NaN stays NaN there; cf. below)
}

// one thread per query row; candidates streamed through a shared-memory tile;
// sorted top-k list (d2, j) with strict '<' insertion: equal distances keep
// the lower index, as the stable argsort does
__global__ void __launch_bounds__(kKnnThreads)
    k_knn_topk(int64_t n, int d, int k, const double *__restrict__ X, const double *__restrict__ sq,
               int64_t *__restrict__ nbr) {
  __shared__ double tile[kKnnTileDoubles];
  __shared__ double tsq[kKnnThreads * 4];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < n;
  double bd[kKnnMaxK];
  int64_t bj[kKnnMaxK];
  for (int t = 0; t < k; ++t) {
    bd[t] = INFINITY;
    bj[t] = INT64_MAX;
  }
  int cnt = 0;
  const double sqi = live ? sq[i] : 0.0;
  const int tp = min(kKnnTileDoubles / d, kKnnThreads * 4);  // candidates per tile
  for (int64_t j0 = 0; j0 < n; j0 += tp) {
    const int nt = (int)min((int64_t)tp, n - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * d; e += blockDim.x) tile[e] = X[j0 * d + e];
    for (int e = threadIdx.x; e < nt; e += blockDim.x) tsq[e] = sq[j0 + e];
    __syncthreads();
    if (!live) continue;
    const double *xi = X + i * d;
    for (int u = 0; u < nt; ++u) {
      const int64_t j = j0 + u;
      if (j == i) continue;  // np.fill_diagonal(d2, inf)
      const double v = pair_d2(xi, tile + (size_t)u * d, d, sqi, tsq[u]);
      // argsort puts NaN last: never better than a number
      if (cnt < k || v < bd[k - 1]) {
        int p = cnt < k ? cnt : k - 1;
        while (p > 0 && v < bd[p - 1]) {
          bd[p] = bd[p - 1];
          bj[p] = bj[p - 1];
          --p;
        }
        bd[p] = v;
        bj[p] = j;
        if (cnt < k) ++cnt;
      } else if (cnt < k) {
        bd[cnt] = v;
        bj[cnt] = j;
        ++cnt;
      }
    }
  }
  if (live)
    for (int t = 0; t < k; ++t) nbr[i * k + t] = bj[t];
}

__global__ void k_knn_keys(int64_t n, int k, const int64_t *__restrict__ nbr,
                           int64_t *__restrict__ key) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k, j = nbr[e];
    key[e] = min(i, j) * n + max(i, j);
  }
}

__global__ void k_knn_edge_d2(int64_t E, int64_t n, int d, const double *__restrict__ X,
                              const double *__restrict__ sq, const int64_t *__restrict__ key,
                              double *__restrict__ d2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = key[e] / n, j = key[e] % n;
    d2[e] = pair_d2(X + i * d, X + j * d, d, sq[i], sq[j]);
  }
}

// numpy's pairwise summation (DOUBLE_pairwise_sum, PW_BLOCKSIZE 128) on one
// thread, so sigma2 is the reference's bit for bit
__device__ double np_pairwise_leaf(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.0;  // numpy: res = 0.; res += a[i] (the -0.0 corner aside)
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int q = 0; q < 8; ++q) r[q] = a[q];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[i + q]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ double np_pairwise(const double *a, int64_t n) {
  if (n <= 128) return np_pairwise_leaf(a, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

__global__ void k_np_pairwise_sum(const double *__restrict__ a, int64_t n, double *__restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = np_pairwise(a, n);
}

// both half-edges of every pair: key (row * n + col), weight
__global__ void k_knn_halves(int64_t E, int64_t n, const int64_t *__restrict__ key,
                             const double *__restrict__ d2, double sigma2, int weighted,
                             int64_t *__restrict__ hkey, double *__restrict__ hw,
                             int64_t *__restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = key[e] / n, j = key[e] % n;
    double w = 1.0;
    if (weighted && sigma2 > 0.0) w = exp(__ddiv_rn(-d2[e], sigma2));
    if (!(w > 0.0) || !isfinite(w)) atomicMin(reinterpret_cast<unsigned long long *>(bad),
                                              (unsigned long long)e);
    hkey[2 * e] = i * n + j;
    hkey[2 * e + 1] = j * n + i;
    hw[2 * e] = w;
    hw[2 * e + 1] = w;
  }
}

__global__ void k_knn_csr(int64_t m, int64_t n, const int64_t *__restrict__ hkey,
                          int64_t *__restrict__ indptr, int64_t *__restrict__ indices) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = hkey[e] / n;
    if (indices) indices[e] = hkey[e] % n;
    // first half-edge of row r (and of the empty rows before it) sets indptr
    const int64_t rp = e ? hkey[e - 1] / n : -1;
    for (int64_t q = rp + 1; q <= r; ++q) indptr[q] = e;
    if (e == m - 1)
      for (int64_t q = r + 1; q <= n; ++q) indptr[q] = m;
  }
}

}  // namespace

KnnResult knn_graph(mg_ctx *ctx, int64_t n, int d, const double *X, int k, bool weighted) {
  require(d >= 1, MG_ERR_INPUT, "feature matrix must be 2-D");
  require(k >= 1 && k < n, MG_ERR_INPUT,
          "k must satisfy 1 <= k < n, got k=" + std::to_string(k) + ", n=" + std::to_string(n));
  require(k <= kKnnMaxK && d <= kKnnTileDoubles, MG_ERR_INPUT,
          "device knn_graph supports k <= 64 and d <= 5120");
  cudaStream_t st = ctx->stream;
  KnnResult r;
  DBuf<double> sq(ctx, n);
  k_knn_sq<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, st>>>(n, d, X, sq.p);
  MG_CHECK_LAUNCH(ctx);
  const int64_t nk = n * k;
  DBuf<int64_t> nbr(ctx, nk), key(ctx, nk), key2(ctx, nk), ne(ctx, 1);
  k_knn_topk<<<(unsigned)((n + kKnnThreads - 1) / kKnnThreads), kKnnThreads, 0, st>>>(n, d, k, X,
                                                                                   sq.p, nbr.p);
  MG_CHECK_LAUNCH(ctx);
  k_knn_keys<<<grid_for(nk, 256, ctx->num_sms * 8), 256, 0, st>>>(n, k, nbr.p, key.p);
  MG_CHECK_LAUNCH(ctx);
  size_t tb1 = 0, tb2 = 0;
  MG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb1, key.p, key2.p, nk, 0, 64, st));
  MG_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, key2.p, key.p, ne.p, nk, st));
  DBuf<unsigned char> tmp(ctx, std::max(tb1, tb2));
  MG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb1, key.p, key2.p, nk, 0, 64, st));
  MG_CUDA(cub::DeviceSelect::Unique(tmp.p, tb2, key2.p, key.p, ne.p, nk, st));
  int64_t E = 0;
  d2h_sync(ctx, &E, ne.p, sizeof(int64_t));
  DBuf<double> d2(ctx, E > 0 ? E : 1), s(ctx, 1);
  k_knn_edge_d2<<<grid_for(E, 256, ctx->num_sms * 8), 256, 0, st>>>(E, n, d, X, sq.p, key.p, d2.p);
  MG_CHECK_LAUNCH(ctx);
  double sigma2 = 1.0;
  if (weighted) {
    k_np_pairwise_sum<<<1, 32, 0, st>>>(d2.p, E, s.p);
    MG_CHECK_LAUNCH(ctx);
    double sum;
    d2h_sync(ctx, &sum, s.p, sizeof(double));
    sigma2 = sum / (double)E;  // dist2.mean()
  }
  r.sigma2 = sigma2;
  const int64_t m = 2 * E;
  DBuf<int64_t> hk(ctx, m), hk2(ctx, m), bad(ctx, 1);
  DBuf<double> hw(ctx, m);
  r.weights.alloc(ctx, m);
  MG_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(int64_t), st));
  k_knn_halves<<<grid_for(E, 256, ctx->num_sms * 8), 256, 0, st>>>(E, n, key.p, d2.p, sigma2,
                                                                   weighted ? 1 : 0, hk.p, hw.p,
                                                                   bad.p);
  MG_CHECK_LAUNCH(ctx);
  int64_t b = -1;
  d2h_sync(ctx, &b, bad.p, sizeof(int64_t));
  if (b >= 0) {  // from_edges: the first offending pair in sorted order
    int64_t kk;
    double dv;
    d2h_sync(ctx, &kk, key.p + b, sizeof(int64_t));
    d2h_sync(ctx, &dv, d2.p + b, sizeof(double));
    const double w = (weighted && sigma2 > 0.0) ? std::exp(-dv / sigma2) : 1.0;
    throw Error(MG_ERR_INPUT, "edge (" + std::to_string(kk / n) + ", " + std::to_string(kk % n) +
                                  ") has non-positive weight " + std::to_string(w));
  }
  size_t tb3 = 0;
  MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb3, hk.p, hk2.p, hw.p, r.weights.p, m, 0, 64, st));
  DBuf<unsigned char> tmp2(ctx, tb3);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp2.p, tb3, hk.p, hk2.p, hw.p, r.weights.p, m, 0, 64, st));
  r.indptr.alloc(ctx, n + 1);
  r.indices.alloc(ctx, m > 0 ? m : 1);
  MG_CUDA(cudaMemsetAsync(r.indptr.p, 0, (n + 1) * sizeof(int64_t), st));
  if (m > 0) {
    k_knn_csr<<<grid_for(m, 256, ctx->num_sms * 8), 256, 0, st>>>(m, n, hk2.p, r.indptr.p,
                                                                  r.indices.p);
    MG_CHECK_LAUNCH(ctx);
  }
  r.nnz = m;
  sync(ctx);
  return r;
}

}  // namespace mg
