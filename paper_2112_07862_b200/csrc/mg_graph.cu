// Operator construction on the device: components, Laplacian, two-hop sets,
// two-hop Laplacian Q, assembly of A = (L - mu Q) + eps I, Gershgorin radii,
// degree balancing.  Reference: /root/reference/pkg/src/manigraph/
// {graph.py, operators.py, sparse.py}; each kernel cites the lines it
// replaces.  Bit-exactness rules: every per-row sum is accumulated
// sequentially in stored (ascending column) order -- the order np.bincount
// uses -- and every product/difference that the reference rounds separately
// is written with __dmul_rn/__dsub_rn/__dadd_rn so nvcc cannot contract it
// into an FMA.
#include <climits>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "mg_graph.cuh"

namespace mg {

static constexpr int kBlock = 256;

// ------------------------------------------------------------ reductions ---
// Deterministic fp64 sum: block b sums the fixed chunk [b*chunk, ...) with a
// fixed tree, then one block sums the partials in order.
__global__ void k_partial_sum(const double *__restrict__ x, int64_t n, int64_t chunk,
                              double *__restrict__ part) {
  __shared__ double sm[kBlock];
  int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += x[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_final_sum(const double *__restrict__ part, int np, double *out) {
  __shared__ double sm[kBlock];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

double sum_f64(mg_ctx *ctx, const double *x, int64_t n) {
  if (n <= 0) return 0.0;
  int nb = grid_for(n, kBlock * 8, 1024);
  int64_t chunk = (n + nb - 1) / nb;
  DBuf<double> part(ctx, nb + 1);
  k_partial_sum<<<nb, kBlock, 0, ctx->stream>>>(x, n, chunk, part.p);
  MG_CHECK_LAUNCH(ctx);
  k_final_sum<<<1, kBlock, 0, ctx->stream>>>(part.p, nb, part.p + nb);
  MG_CHECK_LAUNCH(ctx);
  double r;
  d2h_sync(ctx, &r, part.p + nb, sizeof(double));
  return r;
}

// (value, index) argmin with first-index tie break (np.argmin semantics)
struct VI {
  double v;
  int64_t i;
};
__device__ __forceinline__ VI vi_min(VI a, VI b) {
  if (b.v < a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__global__ void k_partial_argmin(const double *__restrict__ x, int64_t n, int64_t chunk,
                                 VI *__restrict__ part, const int64_t *__restrict__ imap) {
  __shared__ VI sm[kBlock];
  int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  VI best{INFINITY, LLONG_MAX};
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    best = vi_min(best, VI{x[i], imap ? imap[i] : i});
  sm[threadIdx.x] = best;
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = vi_min(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_final_argmin(const VI *__restrict__ part, int np, VI *out) {
  __shared__ VI sm[kBlock];
  VI best{INFINITY, LLONG_MAX};
  for (int i = threadIdx.x; i < np; i += blockDim.x) best = vi_min(best, part[i]);
  sm[threadIdx.x] = best;
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = vi_min(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

static VI argmin_f64(mg_ctx *ctx, const double *x, int64_t n, const int64_t *imap = nullptr) {
  int nb = grid_for(n, kBlock * 8, 1024);
  int64_t chunk = (n + nb - 1) / nb;
  DBuf<VI> part(ctx, nb + 1);
  k_partial_argmin<<<nb, kBlock, 0, ctx->stream>>>(x, n, chunk, part.p, imap);
  MG_CHECK_LAUNCH(ctx);
  k_final_argmin<<<1, kBlock, 0, ctx->stream>>>(part.p, nb, part.p + nb);
  MG_CHECK_LAUNCH(ctx);
  VI r;
  d2h_sync(ctx, &r, part.p + nb, sizeof(VI));
  return r;
}

// ------------------------------------------------------------ components ---
// graph.py:107-123.  Union-find with min-root linking: the final root of a
// component is its smallest node id, so ranking roots by id reproduces the
// reference's DFS-scan label numbering.
__device__ __forceinline__ int uf_find(volatile int *parent, int x) {
  int p = parent[x];
  while (p != x) {
    int gp = parent[p];
    if (gp != p) parent[x] = gp;  // path halving (benign race)
    x = p;
    p = gp;
  }
  return x;
}

__global__ void k_uf_init(int *parent, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = (int)i;
}

__global__ void k_uf_hook(int *parent, int64_t n, const int64_t *__restrict__ ptr,
                          const int64_t *__restrict__ idx) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
      int v = (int)idx[e];
      if (v <= u) continue;
      int a = uf_find(parent, (int)u), b = uf_find(parent, v);
      while (a != b) {
        if (a < b) { int t = a; a = b; b = t; }
        int old = atomicCAS(parent + a, a, b);
        if (old == a) break;
        a = uf_find(parent, old);
        b = uf_find(parent, b);
      }
    }
  }
}

__global__ void k_uf_flatten(int *parent, int64_t n, int64_t *is_root) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = uf_find(parent, (int)i);
    parent[i] = r;
    is_root[i] = (r == (int)i) ? 1 : 0;
  }
}

__global__ void k_uf_label(const int *parent, int64_t n, const int64_t *rank, int64_t *labels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    labels[i] = rank[parent[i]];
}

int64_t components(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                   int64_t *labels) {
  if (n == 0) return 0;
  require(n < INT_MAX, MG_ERR_INPUT, "graph too large for 32-bit node ids");
  DBuf<int> parent(ctx, n);
  DBuf<int64_t> flag(ctx, n + 1), rank(ctx, n + 1);
  int g = grid_for(n, kBlock, ctx->num_sms * 16);
  k_uf_init<<<g, kBlock, 0, ctx->stream>>>(parent.p, n);
  MG_CHECK_LAUNCH(ctx);
  k_uf_hook<<<g, kBlock, 0, ctx->stream>>>(parent.p, n, ptr, idx);
  MG_CHECK_LAUNCH(ctx);
  MG_CUDA(cudaMemsetAsync(flag.p + n, 0, sizeof(int64_t), ctx->stream));
  k_uf_flatten<<<g, kBlock, 0, ctx->stream>>>(parent.p, n, flag.p);
  MG_CHECK_LAUNCH(ctx);
  int64_t count = exclusive_scan_i64(ctx, flag.p, rank.p, n);
  if (labels) {
    k_uf_label<<<g, kBlock, 0, ctx->stream>>>(parent.p, n, rank.p, labels);
    MG_CHECK_LAUNCH(ctx);
  }
  return count;
}

// ------------------------------------------------------------- Laplacian ---
// graph.py:321-346 (degrees: graph.py:93-96, sequential in neighbour order).
__global__ void k_laplacian(int64_t n, const int64_t *__restrict__ ptr,
                            const int64_t *__restrict__ idx, const double *__restrict__ w,
                            int64_t *__restrict__ optr, int64_t *__restrict__ oidx,
                            double *__restrict__ odata) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = ptr[i], e = ptr[i + 1];
    double deg = 0.0;
    for (int64_t k = s; k < e; ++k) deg = __dadd_rn(deg, w[k]);
    int64_t o = s + i;  // out row start = ptr[i] + i
    optr[i] = o;
    if (i == n - 1) optr[n] = e + n;
    bool placed = false;
    for (int64_t k = s; k < e; ++k) {
      int64_t j = idx[k];
      if (!placed && j > i) {
        oidx[o] = i;
        odata[o] = deg;
        ++o;
        placed = true;
      }
      oidx[o] = j;
      odata[o] = -w[k];
      ++o;
    }
    if (!placed) {
      oidx[o] = i;
      odata[o] = deg;
    }
  }
}

void laplacian(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *w,
               int64_t *optr, int64_t *oidx, double *odata) {
  if (n == 0) {
    MG_CUDA(cudaMemsetAsync(optr, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  k_laplacian<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(
      n, ptr, idx, w, optr, oidx, odata);
  MG_CHECK_LAUNCH(ctx);
}

// ----------------------------------------------------------- two-hop sets ---
// operators.py:88-108.  T_i = sorted(unique(U_{m in N(i)} N(m)) \ ({i} U N(i))).
// Rows with <= kWarpCap path products are gathered, bitonic-sorted and
// filtered by one warp in shared memory; larger rows go through a global
// segmented sort.
static constexpr int kWarpCap = 512;
static constexpr int kTHWarps = 8;

__global__ void k_products(int64_t n, const int64_t *__restrict__ ptr,
                           const int64_t *__restrict__ idx, int64_t *__restrict__ prod) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = 0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      int64_t m = idx[k];
      p += ptr[m + 1] - ptr[m];
    }
    prod[i] = p;
  }
}

__device__ __forceinline__ bool in_sorted(const int64_t *__restrict__ a, int64_t lo, int64_t hi,
                                          int64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    int64_t x = a[mid];
    if (x == v) return true;
    if (x < v) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

template <bool FILL>
__global__ void __launch_bounds__(kTHWarps * 32)
    k_two_hop_warp(int64_t n, const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                   const int64_t *__restrict__ prod, int64_t *__restrict__ cnt,
                   const int64_t *__restrict__ tptr, int64_t *__restrict__ tidx) {
  __shared__ int buf[kTHWarps][kWarpCap];
  const unsigned full = 0xffffffffu;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int *b = buf[warp];
  for (int64_t i = (int64_t)blockIdx.x * kTHWarps + warp; i < n;
       i += (int64_t)gridDim.x * kTHWarps) {
    int64_t p = prod[i];
    if (p > kWarpCap) continue;  // large tier
    if (p == 0) {
      if (!FILL && lane == 0) cnt[i] = 0;
      continue;
    }
    int size = 32;
    while (size < p) size <<= 1;
    for (int t = lane; t < size; t += 32) b[t] = INT_MAX;
    __syncwarp();
    int64_t s = ptr[i], e = ptr[i + 1];
    int base = 0;
    for (int64_t c = s; c < e; c += 32) {
      int64_t k = c + lane;
      int d = 0;
      int64_t ms = 0;
      if (k < e) {
        int64_t m = idx[k];
        ms = ptr[m];
        d = (int)(ptr[m + 1] - ms);
      }
      int incl = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += y;
      }
      int off = base + incl - d;
      for (int q = 0; q < d; ++q) b[off + q] = (int)idx[ms + q];
      base += __shfl_sync(full, incl, 31);
    }
    __syncwarp();
    for (int kk = 2; kk <= size; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int t = lane; t < size; t += 32) {
          int partner = t ^ j;
          if (partner > t) {
            int a = b[t], c2 = b[partner];
            bool up = (t & kk) == 0;
            if ((a > c2) == up) {
              b[t] = c2;
              b[partner] = a;
            }
          }
        }
        __syncwarp();
      }
    }
    int64_t out_base = FILL ? tptr[i] : 0;
    int running = 0;
    for (int t0 = 0; t0 < size; t0 += 32) {
      int t = t0 + lane;
      int v = b[t];
      bool keep = v != INT_MAX && (t == 0 || b[t - 1] != v) && (int64_t)v != i;
      if (keep) keep = !in_sorted(idx, s, e, v);
      unsigned mask = __ballot_sync(full, keep);
      if (FILL && keep) tidx[out_base + running + __popc(mask & ((1u << lane) - 1u))] = v;
      running += __popc(mask);
    }
    if (!FILL && lane == 0) cnt[i] = running;
    __syncwarp();
  }
}

__global__ void k_flag_large(int64_t n, const int64_t *__restrict__ prod, int64_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = prod[i] > kWarpCap ? 1 : 0;
}

__global__ void k_list_large(int64_t n, const int64_t *__restrict__ flag,
                             const int64_t *__restrict__ pos, const int64_t *__restrict__ prod,
                             int64_t *rows, int64_t *lprod) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      rows[pos[i]] = i;
      lprod[pos[i]] = prod[i];
    }
}

__global__ void k_gather_large(int64_t nl, const int64_t *__restrict__ rows,
                               const int64_t *__restrict__ off, const int64_t *__restrict__ ptr,
                               const int64_t *__restrict__ idx, int *__restrict__ scratch) {
  for (int64_t r = blockIdx.x; r < nl; r += gridDim.x) {
    int64_t i = rows[r];
    int64_t o = off[r];
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      int64_t m = idx[k];
      int64_t ms = ptr[m], d = ptr[m + 1] - ms;
      for (int64_t q = threadIdx.x; q < d; q += blockDim.x) scratch[o + q] = (int)idx[ms + q];
      o += d;
    }
  }
}

template <bool FILL>
__global__ void k_filter_large(int64_t nl, const int64_t *__restrict__ rows,
                               const int64_t *__restrict__ off, const int *__restrict__ sorted,
                               const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                               int64_t *__restrict__ cnt, const int64_t *__restrict__ tptr,
                               int64_t *__restrict__ tidx) {
  using Scan = cub::BlockScan<int, kBlock>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t running;
  for (int64_t r = blockIdx.x; r < nl; r += gridDim.x) {
    int64_t i = rows[r];
    int64_t lo = off[r], hi = off[r + 1];
    if (threadIdx.x == 0) running = 0;
    __syncthreads();
    for (int64_t c = lo; c < hi; c += kBlock) {
      int64_t t = c + threadIdx.x;
      int keep = 0;
      int v = 0;
      if (t < hi) {
        v = sorted[t];
        keep = (t == lo || sorted[t - 1] != v) && (int64_t)v != i &&
               !in_sorted(idx, ptr[i], ptr[i + 1], v);
      }
      int excl, total;
      Scan(tmp).ExclusiveSum(keep, excl, total);
      if (FILL && keep) tidx[tptr[i] + running + excl] = v;
      __syncthreads();
      if (threadIdx.x == 0) running += total;
      __syncthreads();
    }
    if (!FILL && threadIdx.x == 0) cnt[i] = running;
    __syncthreads();
  }
}

static void two_hop_pass(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                         int64_t *cnt, const int64_t *tptr, int64_t *tidx, bool fill) {
  DBuf<int64_t> prod(ctx, n);
  int g = grid_for(n, kBlock, ctx->num_sms * 16);
  k_products<<<g, kBlock, 0, ctx->stream>>>(n, ptr, idx, prod.p);
  MG_CHECK_LAUNCH(ctx);
  int gw = grid_for(n, kTHWarps, ctx->num_sms * 32);
  if (fill)
    k_two_hop_warp<true><<<gw, kTHWarps * 32, 0, ctx->stream>>>(n, ptr, idx, prod.p, cnt, tptr,
                                                                 tidx);
  else
    k_two_hop_warp<false><<<gw, kTHWarps * 32, 0, ctx->stream>>>(n, ptr, idx, prod.p, cnt, tptr,
                                                                  tidx);
  MG_CHECK_LAUNCH(ctx);
  // large tier
  DBuf<int64_t> flag(ctx, n + 1), pos(ctx, n + 1);
  MG_CUDA(cudaMemsetAsync(flag.p + n, 0, sizeof(int64_t), ctx->stream));
  k_flag_large<<<g, kBlock, 0, ctx->stream>>>(n, prod.p, flag.p);
  MG_CHECK_LAUNCH(ctx);
  int64_t nl = exclusive_scan_i64(ctx, flag.p, pos.p, n);
  if (nl == 0) return;
  DBuf<int64_t> rows(ctx, nl), lprod(ctx, nl + 1), off(ctx, nl + 1);
  MG_CUDA(cudaMemsetAsync(lprod.p + nl, 0, sizeof(int64_t), ctx->stream));
  k_list_large<<<g, kBlock, 0, ctx->stream>>>(n, flag.p, pos.p, prod.p, rows.p, lprod.p);
  MG_CHECK_LAUNCH(ctx);
  int64_t total = exclusive_scan_i64(ctx, lprod.p, off.p, nl);
  DBuf<int> keys(ctx, total), sorted(ctx, total);
  k_gather_large<<<grid_for(nl, 1, 65535), kBlock, 0, ctx->stream>>>(nl, rows.p, off.p, ptr, idx,
                                                                      keys.p);
  MG_CHECK_LAUNCH(ctx);
  size_t tmp = 0;
  MG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, keys.p, sorted.p, total, nl, off.p,
                                             off.p + 1, ctx->stream));
  DBuf<char> t(ctx, tmp);
  MG_CUDA(cub::DeviceSegmentedSort::SortKeys(t.p, tmp, keys.p, sorted.p, total, nl, off.p,
                                             off.p + 1, ctx->stream));
  ctx->launches++;
  if (fill)
    k_filter_large<true><<<grid_for(nl, 1, 65535), kBlock, 0, ctx->stream>>>(
        nl, rows.p, off.p, sorted.p, ptr, idx, cnt, tptr, tidx);
  else
    k_filter_large<false><<<grid_for(nl, 1, 65535), kBlock, 0, ctx->stream>>>(
        nl, rows.p, off.p, sorted.p, ptr, idx, cnt, tptr, tidx);
  MG_CHECK_LAUNCH(ctx);
}

int64_t two_hop_count(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                      int64_t *tptr) {
  if (n == 0) {
    MG_CUDA(cudaMemsetAsync(tptr, 0, sizeof(int64_t), ctx->stream));
    return 0;
  }
  require(n < INT_MAX, MG_ERR_INPUT, "graph too large for 32-bit node ids");
  DBuf<int64_t> cnt(ctx, n + 1);
  MG_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(int64_t), ctx->stream));
  two_hop_pass(ctx, n, ptr, idx, cnt.p, nullptr, nullptr, false);
  return exclusive_scan_i64(ctx, cnt.p, tptr, n);
}

void two_hop_fill(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                  const int64_t *tptr, int64_t *tidx) {
  if (n == 0) return;
  two_hop_pass(ctx, n, ptr, idx, nullptr, tptr, tidx, true);
}

// ------------------------------------------------------ two-hop Laplacian ---
// operators.py:111-135.  inv_i = 1/T_i (0 if empty); Q_ij = -(inv_i + inv_j);
// Q_ii = sequential sum of (inv_i + inv_j) (np.bincount order) or, with
// literal_diagonal, inv_i + (sequential sum of inv_j).
__global__ void k_q_rowlen(int64_t n, const int64_t *__restrict__ tptr, int64_t *len,
                           double *inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = tptr[i + 1] - tptr[i];
    if (len) len[i] = t > 0 ? t + 1 : 0;
    if (inv) inv[i] = t > 0 ? __ddiv_rn(1.0, (double)t) : 0.0;
  }
}

__global__ void k_q_fill(int64_t n, const int64_t *__restrict__ tptr,
                         const int64_t *__restrict__ tidx, const double *__restrict__ inv,
                         int literal, const int64_t *__restrict__ qptr, int64_t *__restrict__ qidx,
                         double *__restrict__ qdata) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = tptr[i], e = tptr[i + 1];
    if (e == s) continue;
    double vi = inv[i];
    double acc = 0.0;
    int64_t o = qptr[i];
    int64_t dpos = -1;
    for (int64_t k = s; k < e; ++k) {
      int64_t j = tidx[k];
      double vj = inv[j];
      double pair = __dadd_rn(vi, vj);
      acc = literal ? __dadd_rn(acc, vj) : __dadd_rn(acc, pair);
      if (dpos < 0 && j > i) dpos = o++;
      qidx[o] = j;
      qdata[o] = -pair;
      ++o;
    }
    if (dpos < 0) dpos = o;
    qidx[dpos] = i;
    qdata[dpos] = literal ? __dadd_rn(vi, acc) : acc;
  }
}

int64_t q_count(mg_ctx *ctx, int64_t n, const int64_t *tptr, int64_t *qptr) {
  if (n == 0) {
    MG_CUDA(cudaMemsetAsync(qptr, 0, sizeof(int64_t), ctx->stream));
    return 0;
  }
  DBuf<int64_t> len(ctx, n + 1);
  MG_CUDA(cudaMemsetAsync(len.p + n, 0, sizeof(int64_t), ctx->stream));
  k_q_rowlen<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(n, tptr, len.p,
                                                                                 nullptr);
  MG_CHECK_LAUNCH(ctx);
  return exclusive_scan_i64(ctx, len.p, qptr, n);
}

void q_fill(mg_ctx *ctx, int64_t n, const int64_t *tptr, const int64_t *tidx, int literal,
            const int64_t *qptr, int64_t *qidx, double *qdata) {
  if (n == 0) return;
  DBuf<double> inv(ctx, n);
  int g = grid_for(n, kBlock, ctx->num_sms * 16);
  k_q_rowlen<<<g, kBlock, 0, ctx->stream>>>(n, tptr, nullptr, inv.p);
  MG_CHECK_LAUNCH(ctx);
  k_q_fill<<<g, kBlock, 0, ctx->stream>>>(n, tptr, tidx, inv.p, literal, qptr, qidx, qdata);
  MG_CHECK_LAUNCH(ctx);
}

// ------------------------------------------------------- symmetry check ---
// sparse.py:100-105: max |M - M^T| over stored entries vs rtol * max(max|M|, 1).
__global__ void k_sym_rows(int64_t n, const int64_t *__restrict__ ptr,
                           const int64_t *__restrict__ idx, const double *__restrict__ data,
                           double *__restrict__ dmax, double *__restrict__ vmax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double dm = 0.0, vm = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      int64_t j = idx[k];
      double v = data[k];
      vm = fmax(vm, fabs(v));
      // find (j, i)
      int64_t lo = ptr[j], hi = ptr[j + 1];
      double vt = 0.0;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        int64_t x = idx[mid];
        if (x == i) { vt = data[mid]; break; }
        if (x < i) lo = mid + 1;
        else hi = mid;
      }
      dm = fmax(dm, fabs(__dsub_rn(v, vt)));
    }
    dmax[i] = dm;
    vmax[i] = vm;
  }
}

__global__ void k_neg_inplace(double *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = -x[i];
}

static double max_f64(mg_ctx *ctx, double *x, int64_t n) {
  // max via argmin of the negation (x >= 0 here)
  k_neg_inplace<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(x, n);
  MG_CHECK_LAUNCH(ctx);
  VI r = argmin_f64(ctx, x, n);
  return -r.v;
}

double max_f64_const(mg_ctx *ctx, const double *x, int64_t n) {
  if (n <= 0) return -INFINITY;
  DBuf<double> t(ctx, n);
  MG_CUDA(cudaMemcpyAsync(t.p, x, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  k_neg_inplace<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(t.p, n);
  MG_CHECK_LAUNCH(ctx);
  VI r = argmin_f64(ctx, t.p, n);
  return -r.v;
}

bool check_symmetric(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                     const double *data, double rtol) {
  if (n == 0) return true;
  DBuf<double> dm(ctx, n), vm(ctx, n);
  k_sym_rows<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(n, ptr, idx, data,
                                                                                 dm.p, vm.p);
  MG_CHECK_LAUNCH(ctx);
  double dmax = max_f64(ctx, dm.p, n);
  double scale = max_f64(ctx, vm.p, n);
  return !(dmax > rtol * fmax(scale, 1.0));
}

// ------------------------------------------------------ repulsion weight ---
// operators.py:159-176: mu = min_{Q_ii > 0} eps / (2 Q_ii - rowsum_i).
__global__ void k_mu_rows(int64_t n, const int64_t *__restrict__ ptr,
                          const int64_t *__restrict__ idx, const double *__restrict__ data,
                          double eps, double *__restrict__ crit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0, rs = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      rs = __dadd_rn(rs, data[k]);
      if (idx[k] == i) d = data[k];
    }
    double c = INFINITY;
    if (d > 0.0) {
      double den = __dsub_rn(__dmul_rn(2.0, d), rs);
      c = __ddiv_rn(eps, den);
      if (c != c) c = -INFINITY;  // NaN propagates through np.min: flag it
    }
    crit[i] = c;
  }
}

double repulsion_weight(mg_ctx *ctx, int64_t n, const int64_t *qptr, const int64_t *qidx,
                        const double *qdata, double eps) {
  require(eps >= 0.0, MG_ERR_INPUT, "epsilon must be non-negative, got " + std::to_string(eps));
  if (n == 0) return 0.0;
  DBuf<double> crit(ctx, n);
  k_mu_rows<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(n, qptr, qidx,
                                                                                 qdata, eps, crit.p);
  MG_CHECK_LAUNCH(ctx);
  VI r = argmin_f64(ctx, crit.p, n);
  if (r.v == INFINITY) return 0.0;  // no row with Q_ii > 0
  if (r.v == -INFINITY) return NAN;
  return r.v;
}

// ------------------------------------------------------------- assembly ---
// operators.py:179-186.  scipy evaluates r1 = L - (mu*Q) over the union
// pattern (dropping exact zeros), then r1 + eps*I (dropping zeros again).
// Per entry: A_ij = fl(fl(L_ij - fl(mu*Q_ij)) + [i==j] eps), absent = 0.
template <bool FILL>
__global__ void k_assemble(int64_t n, const int64_t *__restrict__ lptr,
                           const int64_t *__restrict__ lidx, const double *__restrict__ ldata,
                           const int64_t *__restrict__ qptr, const int64_t *__restrict__ qidx,
                           const double *__restrict__ qdata, double mu, double eps,
                           int64_t *__restrict__ cnt, const int64_t *__restrict__ aptr,
                           int64_t *__restrict__ aidx, double *__restrict__ adata) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = lptr[i], ae = lptr[i + 1], b = qptr[i], be = qptr[i + 1];
    bool diag_done = false;
    int64_t o = FILL ? aptr[i] : 0;
    int64_t c = 0;
    while (true) {
      int64_t ca = a < ae ? lidx[a] : LLONG_MAX;
      int64_t cb = b < be ? qidx[b] : LLONG_MAX;
      int64_t cd = diag_done ? LLONG_MAX : i;
      int64_t col = min(ca, min(cb, cd));
      if (col == LLONG_MAX) break;
      double lv = 0.0, qv = 0.0;
      if (ca == col) lv = ldata[a++];
      if (cb == col) qv = qdata[b++];
      double r1 = __dsub_rn(lv, __dmul_rn(mu, qv));
      double v = r1;
      if (col == i) {
        v = __dadd_rn(r1, eps);
        diag_done = true;
      }
      if (v != 0.0) {
        if (FILL) {
          aidx[o] = col;
          adata[o] = v;
          ++o;
        }
        ++c;
      }
    }
    if (!FILL) cnt[i] = c;
  }
}

int64_t assemble_count(mg_ctx *ctx, int64_t n, const int64_t *lptr, const int64_t *lidx,
                       const double *ldata, const int64_t *qptr, const int64_t *qidx,
                       const double *qdata, double mu, double eps, int64_t *aptr) {
  if (n == 0) {
    MG_CUDA(cudaMemsetAsync(aptr, 0, sizeof(int64_t), ctx->stream));
    return 0;
  }
  DBuf<int64_t> cnt(ctx, n + 1);
  MG_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(int64_t), ctx->stream));
  k_assemble<false><<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(
      n, lptr, lidx, ldata, qptr, qidx, qdata, mu, eps, cnt.p, nullptr, nullptr, nullptr);
  MG_CHECK_LAUNCH(ctx);
  return exclusive_scan_i64(ctx, cnt.p, aptr, n);
}

void assemble_fill(mg_ctx *ctx, int64_t n, const int64_t *lptr, const int64_t *lidx,
                   const double *ldata, const int64_t *qptr, const int64_t *qidx,
                   const double *qdata, double mu, double eps, const int64_t *aptr,
                   int64_t *aidx, double *adata) {
  if (n == 0) return;
  k_assemble<true><<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(
      n, lptr, lidx, ldata, qptr, qidx, qdata, mu, eps, nullptr, aptr, aidx, adata);
  MG_CHECK_LAUNCH(ctx);
}

// ------------------------------------------------------ degree balancing ---
// sparse.py:84-94 (radii, sequential), operators.py:189-219 (log space,
// two mean passes).
__global__ void k_radii(int64_t n, const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                        const double *__restrict__ data, double *__restrict__ radius,
                        double *__restrict__ left, unsigned long long *first_bad,
                        const int64_t *__restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double r = 0.0, d = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      if (idx[k] == i) d = data[k];
      else r = __dadd_rn(r, fabs(data[k]));
    }
    if (radius) radius[i] = r;
    if (left) left[i] = __dsub_rn(d, r);
    if (first_bad && !(r > 0.0)) atomicMin(first_bad, (unsigned long long)(perm ? perm[i] : i));
  }
}

int64_t degree_balancing(mg_ctx *ctx, int64_t n, const int64_t *aptr, const int64_t *aidx,
                         const double *adata, double *b, double *gdeg, const int64_t *perm) {
  if (n == 0) {
    *gdeg = NAN;
    return -1;
  }
  DBuf<double> rad(ctx, n);
  DBuf<unsigned long long> bad(ctx, 1);
  MG_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), ctx->stream));
  int g = grid_for(n, kBlock, ctx->num_sms * 16);
  k_radii<<<g, kBlock, 0, ctx->stream>>>(n, aptr, aidx, adata, rad.p, nullptr, bad.p, perm);
  MG_CHECK_LAUNCH(ctx);
  unsigned long long first;
  d2h_sync(ctx, &first, bad.p, sizeof(first));
  if (first != ~0ull) return (int64_t)first;
  // means as numpy's pairwise sums (np.mean), mg_queries.cu
  balance_radii(ctx, n, rad.p, b, gdeg, perm);
  return -1;
}

void disc_left_min(mg_ctx *ctx, int64_t n, const int64_t *aptr, const int64_t *aidx,
                   const double *adata, double *min_left, int64_t *row, const int64_t *perm) {
  if (n == 0) {
    *min_left = NAN;
    *row = 0;
    return;
  }
  DBuf<double> left(ctx, n);
  k_radii<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(
      n, aptr, aidx, adata, nullptr, left.p, nullptr, nullptr);
  MG_CHECK_LAUNCH(ctx);
  VI r = argmin_f64(ctx, left.p, n, perm);
  *min_left = r.v;
  *row = r.i;
}

__global__ void k_diag(int64_t n, const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                       const double *__restrict__ data, double *__restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
      if (idx[k] == i) v = data[k];
    d[i] = v;
  }
}

double trace(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *data) {
  if (n == 0) return 0.0;
  DBuf<double> d(ctx, n);
  k_diag<<<grid_for(n, kBlock, ctx->num_sms * 16), kBlock, 0, ctx->stream>>>(n, ptr, idx, data,
                                                                             d.p);
  MG_CHECK_LAUNCH(ctx);
  return sum_f64(ctx, d.p, n);
}

}  // namespace mg
