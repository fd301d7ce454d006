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
// Search (round 2): for d <= 3 and n >= 4096 a uniform cell grid (about two
// points per cell, points bucketed by a radix sort of their cell ids) replaces
// the all-pairs scan.  Each query visits Chebyshev shells of cells around its
// own until its k-th candidate is closer than anything outside the visited
// box can be (true distance bound minus a rounding margin for the reference's
// sq_i + sq_j - 2 x.x form), so the top-k lists -- compared as (d2, index)
// pairs, i.e. ties to the lower index -- are exactly the all-pairs ones.
// Small n, larger d or non-finite inputs keep the exact O(n^2 d) scan.
#include <cub/cub.cuh>
#include <vector>

#include "mg_common.cuh"
#include "mg_graph.cuh"
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

// ------------------------------------------------------------- grid search ---
constexpr int kGridMaxD = 3;

struct GridSpec {
  int d;
  int64_t G[kGridMaxD];   // cells per dimension
  double lo[kGridMaxD], h[kGridMaxD];
  double sqmax;
};

__device__ __forceinline__ int64_t cell_coord(double x, int q, const GridSpec &gs) {
  int64_t c = (int64_t)floor((x - gs.lo[q]) / gs.h[q]);
  return c < 0 ? 0 : (c >= gs.G[q] ? gs.G[q] - 1 : c);
}

__global__ void k_bbox(int64_t n, int d, const double *__restrict__ X, double *__restrict__ part) {
  // part[block][2d]: min then max per dimension; also flags non-finite values (NaN -> min)
  __shared__ double smin[kGridMaxD][256], smax[kGridMaxD][256];
  double mn[kGridMaxD], mx[kGridMaxD];
  for (int q = 0; q < d; ++q) {
    mn[q] = INFINITY;
    mx[q] = -INFINITY;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int q = 0; q < d; ++q) {
      const double v = X[i * d + q];
      if (!isfinite(v)) mn[q] = NAN;
      if (!(v >= mn[q])) mn[q] = isnan(mn[q]) ? mn[q] : v;
      if (v > mx[q]) mx[q] = v;
    }
  for (int q = 0; q < d; ++q) {
    smin[q][threadIdx.x] = mn[q];
    smax[q][threadIdx.x] = mx[q];
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < d; ++q) {
      double a = INFINITY, b = -INFINITY;
      for (int t = 0; t < (int)blockDim.x; ++t) {
        const double u = smin[q][t];
        if (isnan(u) || isnan(a)) a = NAN;
        else a = fmin(a, u);
        b = fmax(b, smax[q][t]);
      }
      part[blockIdx.x * 2 * d + q] = a;
      part[blockIdx.x * 2 * d + d + q] = b;
    }
}

__global__ void k_cells(int64_t n, GridSpec gs, const double *__restrict__ X,
                        int64_t *__restrict__ cell, int64_t *__restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int q = gs.d - 1; q >= 0; --q) c = c * gs.G[q] + cell_coord(X[i * gs.d + q], q, gs);
    cell[i] = c;
    id[i] = i;
  }
}

// start[c] = first sorted position of cell c (start[ncells] = n)
__global__ void k_cell_starts(int64_t n, int64_t ncells, const int64_t *__restrict__ cell,
                              int64_t *__restrict__ start) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cell[p], cp = p ? cell[p - 1] : -1;
    for (int64_t q = cp + 1; q <= c; ++q) start[q] = p;
    if (p == n - 1)
      for (int64_t q = c + 1; q <= ncells; ++q) start[q] = n;
  }
}

__global__ void k_gather_sorted(int64_t n, int d, const int64_t *__restrict__ id,
                                const double *__restrict__ X, const double *__restrict__ sq,
                                double *__restrict__ Xs, double *__restrict__ sqs) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = id[p];
    for (int q = 0; q < d; ++q) Xs[p * d + q] = X[i * d + q];
    sqs[p] = sq[i];
  }
}

// one thread per query (queries in cell order for locality)
template <int D>
__global__ void __launch_bounds__(128)
    k_knn_grid(int64_t n, int k, GridSpec gs, const int64_t *__restrict__ id,
               const double *__restrict__ Xs, const double *__restrict__ sqs,
               const int64_t *__restrict__ start, int64_t *__restrict__ nbr) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t i = id[p];
  double xi[D];
  for (int q = 0; q < D; ++q) xi[q] = Xs[p * D + q];
  const double sqi = sqs[p];
  int64_t ci[D];
  for (int q = 0; q < D; ++q) ci[q] = cell_coord(xi[q], q, gs);
  double bd[kKnnMaxK];
  int64_t bj[kKnnMaxK];
  int cnt = 0;
  // rounding margin of d2 = (sq_i + sq_j) - 2 x_i.x_j against the true squared distance
  const double tol = 64.0 * 2.220446049250313e-16 * (sqi + gs.sqmax + 2.0 * sqrt(sqi * gs.sqmax)) +
                     1e-300;
  int64_t gmax = 0;
  for (int q = 0; q < D; ++q) gmax = max(gmax, gs.G[q]);
  for (int64_t r = 0; r <= gmax; ++r) {
    // cells with Chebyshev distance exactly r from ci, clipped to the grid
    int64_t lo[D], hi[D];
    for (int q = 0; q < D; ++q) {
      lo[q] = max((int64_t)0, ci[q] - r);
      hi[q] = min(gs.G[q] - 1, ci[q] + r);
    }
    int64_t c[D];
    for (int q = 0; q < D; ++q) c[q] = lo[q];
    while (true) {
      bool shell = false;
      for (int q = 0; q < D; ++q) shell |= (c[q] == ci[q] - r) || (c[q] == ci[q] + r);
      if (shell) {
        int64_t lin = 0;
        for (int q = D - 1; q >= 0; --q) lin = lin * gs.G[q] + c[q];
        for (int64_t pp = start[lin]; pp < start[lin + 1]; ++pp) {
          const int64_t j = id[pp];
          if (j == i) continue;
          const double v = pair_d2(xi, Xs + pp * D, D, sqi, sqs[pp]);
          if (cnt < k) {
            int t = cnt++;
            while (t > 0 && (v < bd[t - 1] || (v == bd[t - 1] && j < bj[t - 1]))) {
              bd[t] = bd[t - 1];
              bj[t] = bj[t - 1];
              --t;
            }
            bd[t] = v;
            bj[t] = j;
          } else if (v < bd[k - 1] || (v == bd[k - 1] && j < bj[k - 1])) {
            int t = k - 1;
            while (t > 0 && (v < bd[t - 1] || (v == bd[t - 1] && j < bj[t - 1]))) {
              bd[t] = bd[t - 1];
              bj[t] = bj[t - 1];
              --t;
            }
            bd[t] = v;
            bj[t] = j;
          }
        }
      }
      int q = 0;
      for (; q < D; ++q) {
        if (c[q] < hi[q]) {
          ++c[q];
          break;
        }
        c[q] = lo[q];
      }
      if (q == D) break;
    }
    // everything not yet visited lies outside the box of cells within r of ci:
    // true distance >= the gap from xi to that box's faces (domain edges excluded)
    double safe = INFINITY;
    bool all = true;
    for (int q = 0; q < D; ++q) {
      if (ci[q] - r > 0) {
        safe = fmin(safe, (xi[q] - gs.lo[q]) - (double)(ci[q] - r) * gs.h[q]);
        all = false;
      }
      if (ci[q] + r < gs.G[q] - 1) {
        safe = fmin(safe, (double)(ci[q] + r + 1) * gs.h[q] - (xi[q] - gs.lo[q]));
        all = false;
      }
    }
    if (all) break;
    if (cnt == k && safe > 0.0 && bd[k - 1] < safe * safe - tol) break;
  }
  for (int t = 0; t < k; ++t) nbr[i * k + t] = t < cnt ? bj[t] : i;
}

// true: nbr filled by the grid search; false: not applicable (caller scans all pairs)
bool knn_topk_grid(mg_ctx *ctx, int64_t n, int d, const double *X, const double *sq, int k,
                   int64_t *nbr) {
  const char *env = getenv("MG_KNN_GRID");
  if (env && env[0] == '0') return false;
  if (d < 1 || d > kGridMaxD || n < 4096) return false;
  cudaStream_t st = ctx->stream;
  const int nb = 148;
  DBuf<double> part(ctx, (size_t)nb * 2 * d);
  k_bbox<<<nb, 256, 0, st>>>(n, d, X, part.p);
  MG_CHECK_LAUNCH(ctx);
  std::vector<double> hp((size_t)nb * 2 * d);
  d2h_sync(ctx, hp.data(), part.p, hp.size() * sizeof(double));
  GridSpec gs{};
  gs.d = d;
  double span[kGridMaxD];
  for (int q = 0; q < d; ++q) {
    double a = INFINITY, b = -INFINITY;
    for (int t = 0; t < nb; ++t) {
      const double u = hp[(size_t)t * 2 * d + q];
      if (std::isnan(u)) return false;  // non-finite coordinates: exact scan keeps numpy's NaN order
      a = std::min(a, u);
      b = std::max(b, hp[(size_t)t * 2 * d + d + q]);
    }
    gs.lo[q] = a;
    span[q] = b - a;
  }
  // ~2 points per cell over the non-degenerate dimensions
  int live = 0;
  for (int q = 0; q < d; ++q) live += span[q] > 0.0;
  const double per = live ? std::pow((double)n / 2.0, 1.0 / live) : 1.0;
  int64_t ncells = 1;
  for (int q = 0; q < d; ++q) {
    gs.G[q] = span[q] > 0.0 ? std::max<int64_t>(1, (int64_t)per) : 1;
    gs.h[q] = span[q] > 0.0 ? span[q] / (double)gs.G[q] * (1.0 + 1e-12) : 1.0;
    ncells *= gs.G[q];
  }
  gs.sqmax = max_f64_const(ctx, sq, n);
  DBuf<int64_t> cell(ctx, n), cell2(ctx, n), id(ctx, n), id2(ctx, n), start(ctx, ncells + 1);
  k_cells<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, st>>>(n, gs, X, cell.p, id.p);
  MG_CHECK_LAUNCH(ctx);
  int bits = 1;
  while (bits < 63 && ((int64_t)1 << bits) <= ncells) ++bits;
  size_t tb = 0;
  MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, cell.p, cell2.p, id.p, id2.p, n, 0, bits, st));
  DBuf<unsigned char> tmp(ctx, tb);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, cell.p, cell2.p, id.p, id2.p, n, 0, bits, st));
  ctx->launches++;
  k_cell_starts<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, st>>>(n, ncells, cell2.p, start.p);
  MG_CHECK_LAUNCH(ctx);
  DBuf<double> Xs(ctx, (size_t)n * d), sqs(ctx, n);
  k_gather_sorted<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, st>>>(n, d, id2.p, X, sq, Xs.p,
                                                                      sqs.p);
  MG_CHECK_LAUNCH(ctx);
  const unsigned g = (unsigned)((n + 127) / 128);
  if (d == 1)
    k_knn_grid<1><<<g, 128, 0, st>>>(n, k, gs, id2.p, Xs.p, sqs.p, start.p, nbr);
  else if (d == 2)
    k_knn_grid<2><<<g, 128, 0, st>>>(n, k, gs, id2.p, Xs.p, sqs.p, start.p, nbr);
  else
    k_knn_grid<3><<<g, 128, 0, st>>>(n, k, gs, id2.p, Xs.p, sqs.p, start.p, nbr);
  MG_CHECK_LAUNCH(ctx);
  sync(ctx);
  return true;
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
  if (!knn_topk_grid(ctx, n, d, X, sq.p, k, nbr.p)) {
    k_knn_topk<<<(unsigned)((n + kKnnThreads - 1) / kKnnThreads), kKnnThreads, 0, st>>>(
        n, d, k, X, sq.p, nbr.p);
    MG_CHECK_LAUNCH(ctx);
  }
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
  DBuf<double> d2(ctx, E > 0 ? E : 1);
  k_knn_edge_d2<<<grid_for(E, 256, ctx->num_sms * 8), 256, 0, st>>>(E, n, d, X, sq.p, key.p, d2.p);
  MG_CHECK_LAUNCH(ctx);
  double sigma2 = 1.0;
  if (weighted) {
    sigma2 = np_sum_f64(ctx, d2.p, E) / (double)E;  // dist2.mean(), numpy's pairwise sum
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
