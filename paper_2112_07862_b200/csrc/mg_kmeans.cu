// k-means (k-means++ seeding + Lloyd, best of R restarts) and normalize_rows
// on the device -- clustering.py:50-134 of the reference, with its portable
// xoshiro256** / splitmix64 streams (rng.py:9-127) driven on the host, so the
// seeding draws are the reference's draws.
//
// Per restart (kmeans.py semantics):
//   centers[0] = pts[rng.index(n)];  d2 = |pts - c0|^2
//   for j < c: cum = cumsum(d2); centers[j] = pts[rng.weighted_index(cum)];
//              d2 = min(d2, |pts - cj|^2)
//   Lloyd (<= 300 iterations): labels = argmin_j |x|^2 - 2 x.c_j + |c_j|^2
//   (first minimum), empty clusters repaired by stealing the worst-fit point of
//   a cluster with > 1 member (cluster order), stop when labels repeat,
//   centers = member means; wcss = sum |x - c_label|^2.
// The lowest wcss wins, ties by the lowest restart index.
//
// Device layout: points n x d row-major fp64 (d <= 32, c <= 64).  One warp
// per row for the centroid sums (lane = dimension), accumulated in a fixed
// order (warp rows in sequence, warps then blocks in index order): the
// centers -- and hence the labels -- are run-to-run deterministic.
// Differences from the reference's arithmetic, all at the 1e-16 level: the
// d2 prefix sum is a parallel scan (numpy's cumsum is sequential), the
// centroid sums are block-ordered (numpy's mean is pairwise) and the dot
// products use fused multiply-adds (BLAS dgemm).  A draw or an argmin can
// only change when two candidates tie to that precision.
#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "mg_common.cuh"
#include "mg_kmeans.cuh"

namespace mg {

namespace {

constexpr int kKmMaxD = 32;
constexpr int kKmMaxC = 64;
constexpr int kKmMaxIter = 300;  // clustering.py:21
constexpr int kKmBlocks = 592;   // 4 x 148 SMs
constexpr int kKmThreads = 256;

// ------------------------------------------------------------------ RNG ---
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull, kStream = 0xD2B74407B1CE6E93ull;

uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t stream_seed(uint64_t seed, uint64_t r) { return mix64(mix64(seed) + (r + 1) * kStream); }
uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t z = seed;
    for (int i = 0; i < 4; ++i) {
      z += kGolden;
      s[i] = mix64(z);
    }
    if (!(s[0] | s[1] | s[2] | s[3])) s[0] = 1;
  }
  uint64_t next() {
    const uint64_t out = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  int64_t index(int64_t n) {
    const int64_t i = (int64_t)(uniform() * (double)n);
    return i >= n ? n - 1 : i;
  }
};

// ------------------------------------------------------------- kernels ---
// d2[i] = |x_i - c|^2 (mode 0: set, 1: min with the current value); the
// element order of the sum matches numpy's (x - c)**2 summed along axis 1
__global__ void k_km_d2(int64_t n, int d, const double *__restrict__ X, const double *__restrict__ c,
                        double *__restrict__ d2, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < d; ++q) {
      const double t = __dsub_rn(X[i * d + q], c[q]);
      s = __dadd_rn(s, __dmul_rn(t, t));
    }
    d2[i] = mode ? fmin(d2[i], s) : s;
  }
}

// first index with cum[i] > r (weighted_index's bisection; cum is inclusive)
__global__ void k_km_search(int64_t n, const double *__restrict__ cum, double r,
                            int64_t *__restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (cum[mid] > r) hi = mid;
      else lo = mid + 1;
    }
    *out = lo;
  }
}

__global__ void k_km_gather_row(int d, const double *__restrict__ X, const int64_t *__restrict__ idx,
                                double *__restrict__ dst) {
  for (int q = threadIdx.x; q < d; q += blockDim.x) dst[q] = X[*idx * d + q];
}

// labels = argmin_j (|x|^2 - 2 x.c_j + |c_j|^2); fit = that minimum; counts;
// changed flag.  Centers and |c|^2 staged in shared memory.
__global__ void __launch_bounds__(kKmThreads)
    k_km_assign(int64_t n, int d, int c, const double *__restrict__ X,
                const double *__restrict__ C, const int64_t *__restrict__ old,
                int64_t *__restrict__ lab, double *__restrict__ fit, int *__restrict__ counts,
                int *__restrict__ changed) {
  __shared__ double sC[kKmMaxC * kKmMaxD];
  __shared__ double sq[kKmMaxC];
  __shared__ int scnt[kKmMaxC];
  for (int e = threadIdx.x; e < c * d; e += blockDim.x) sC[e] = C[e];
  for (int j = threadIdx.x; j < c; j += blockDim.x) scnt[j] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < d; ++q) s += sC[j * d + q] * sC[j * d + q];
    sq[j] = s;
  }
  __syncthreads();
  int ch = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x[kKmMaxD];
    double xx = 0.0;
    for (int q = 0; q < d; ++q) {
      x[q] = X[i * d + q];
      xx += x[q] * x[q];
    }
    double best = 0.0;
    int bj = 0;
    for (int j = 0; j < c; ++j) {
      double dot = 0.0;
      for (int q = 0; q < d; ++q) dot += x[q] * sC[j * d + q];
      const double v = xx - 2.0 * dot + sq[j];
      if (j == 0 || v < best) {
        best = v;
        bj = j;
      }
    }
    lab[i] = bj;
    fit[i] = best;
    ch |= (old[i] != bj);
    atomicAdd(&scnt[bj], 1);
  }
  if (ch) atomicOr(changed, 1);
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x)
    if (scnt[j]) atomicAdd(&counts[j], scnt[j]);
}

// fit masked to rows whose cluster keeps > 1 member (clustering.py:76-78)
__global__ void k_km_mask_fit(int64_t n, const int64_t *__restrict__ lab,
                              const double *__restrict__ fit, const int *__restrict__ counts,
                              double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = counts[lab[i]] > 1 ? fit[i] : -INFINITY;
}

// per-block centroid partial sums in a fixed order: warp w of block b sums the
// rows of its contiguous sub-range in sequence (lane = dimension); warps are
// then added in index order.  part[b][j][q], pcnt not needed (counts known).
__global__ void __launch_bounds__(kKmThreads)
    k_km_sums(int64_t n, int d, int c, const double *__restrict__ X,
              const int64_t *__restrict__ lab, double *__restrict__ part) {
  __shared__ double acc[kKmThreads / 32][kKmMaxC * kKmMaxD / 4];  // c * d <= 512 per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kKmThreads / 32;
  for (int e = lane; e < c * d; e += 32) acc[warp][e] = 0.0;
  __syncwarp();
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  const int64_t w0 = r0 + (r1 - r0) * warp / nw, w1 = r0 + (r1 - r0) * (warp + 1) / nw;
  for (int64_t i = w0; i < w1; ++i) {
    const int j = (int)lab[i];
    if (lane < d) acc[warp][j * d + lane] += X[i * d + lane];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < c * d; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[w][e];
    part[(size_t)blockIdx.x * c * d + e] = s;
  }
}

__global__ void k_km_centers(int nb, int d, int c, const double *__restrict__ part,
                             const int *__restrict__ counts, double *__restrict__ C) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < c * d; e += gridDim.x * blockDim.x) {
    const int j = e / d;
    if (counts[j] == 0) continue;  // no members: center kept (clustering.py:90-92)
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(size_t)b * c * d + e];
    C[e] = s / (double)counts[j];
  }
}

__global__ void k_km_wcss(int64_t n, int d, const double *__restrict__ X,
                          const double *__restrict__ C, const int64_t *__restrict__ lab,
                          double *__restrict__ part) {
  __shared__ double red[kKmThreads];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double *c = C + lab[i] * d;
    for (int q = 0; q < d; ++q) {
      const double t = X[i * d + q] - c[q];
      s += t * t;
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_km_diff(int64_t n, const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                          int *__restrict__ changed) {
  int ch = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ch |= a[i] != b[i];
  if (ch) atomicOr(changed, 1);
}

__global__ void k_km_set_label(int64_t *__restrict__ lab, const int64_t *__restrict__ idx,
                               int j, int *__restrict__ counts, int64_t n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t i = *idx;
    if (i < 0 || i >= n) return;
    atomicSub(&counts[lab[i]], 1);
    lab[i] = j;
    atomicAdd(&counts[j], 1);
  }
}

__global__ void k_km_normalize(int64_t n, int d, const double *__restrict__ X,
                               double *__restrict__ Y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < d; ++q) s += X[i * d + q] * X[i * d + q];
    const double nrm = sqrt(s);
    for (int q = 0; q < d; ++q) Y[i * d + q] = nrm > 0.0 ? X[i * d + q] / nrm : X[i * d + q];
  }
}

struct ArgMax {
  __device__ __forceinline__ cub::KeyValuePair<int64_t, double> operator()(
      const cub::KeyValuePair<int64_t, double> &a, const cub::KeyValuePair<int64_t, double> &b) const {
    if (b.value > a.value || (b.value == a.value && b.key < a.key)) return b;
    return a;
  }
};

}  // namespace

void normalize_rows(mg_ctx *ctx, int64_t n, int d, const double *X, double *Y) {
  require(n >= 1 && d >= 1, MG_ERR_INPUT, "points must form a non-empty 2-D array");
  k_km_normalize<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(n, d, X, Y);
  MG_CHECK_LAUNCH(ctx);
}

double kmeans(mg_ctx *ctx, int64_t n, int d, const double *X, int c, int restarts, uint64_t seed,
              int64_t *labels_out) {
  require(n >= 1 && d >= 1, MG_ERR_INPUT, "points must form a non-empty 2-D array");
  require(c >= 1 && c <= n, MG_ERR_INPUT,
          "cluster count must be in [1, " + std::to_string(n) + "], got " + std::to_string(c));
  require(restarts >= 1, MG_ERR_INPUT, "restarts must be >= 1, got " + std::to_string(restarts));
  require(d <= kKmMaxD && c <= kKmMaxC && c * d <= kKmMaxC * kKmMaxD / 4, MG_ERR_INPUT,
          "device k-means supports d <= 32, c <= 64, c*d <= 512");
  cudaStream_t st = ctx->stream;
  if (c == 1 || c == n) {  // clustering.py:119-122
    std::vector<int64_t> h(n);
    for (int64_t i = 0; i < n; ++i) h[i] = c == 1 ? 0 : i;
    MG_CUDA(cudaMemcpyAsync(labels_out, h.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    sync(ctx);
    return 0.0;
  }
  const int g = grid_for(n, kKmThreads, kKmBlocks);
  DBuf<double> d2(ctx, n), cum(ctx, n), fit(ctx, n), C(ctx, (size_t)c * d),
      part(ctx, (size_t)kKmBlocks * c * d), wpart(ctx, kKmBlocks);
  DBuf<int64_t> lab(ctx, n), lab2(ctx, n), sel(ctx, 1);
  DBuf<int> counts(ctx, c), changed(ctx, 1);
  DBuf<cub::KeyValuePair<int64_t, double>> amax(ctx, 1);
  size_t tb_scan = 0, tb_max = 0;
  MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb_scan, d2.p, cum.p, n, st));
  MG_CUDA(cub::DeviceReduce::Reduce(nullptr, tb_max, cub::ArgIndexInputIterator<const double *, int64_t>(fit.p),
                                    amax.p, n, ArgMax(),
                                    cub::KeyValuePair<int64_t, double>(0, -INFINITY), st));
  DBuf<unsigned char> tmp(ctx, std::max(tb_scan, tb_max));
  double best_wcss = 0.0;
  for (int r = 0; r < restarts; ++r) {
    Xoshiro rng(stream_seed(seed, (uint64_t)r));
    // ---- k-means++ seeding (clustering.py:57-67)
    int64_t i0 = rng.index(n);
    MG_CUDA(cudaMemcpyAsync(C.p, X + i0 * d, d * sizeof(double), cudaMemcpyDeviceToDevice, st));
    k_km_d2<<<g, kKmThreads, 0, st>>>(n, d, X, C.p, d2.p, 0);
    MG_CHECK_LAUNCH(ctx);
    for (int j = 1; j < c; ++j) {
      size_t tb = tmp.n;
      MG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, d2.p, cum.p, n, st));
      double total;
      d2h_sync(ctx, &total, cum.p + n - 1, sizeof(double));
      if (total <= 0.0) {  // rng.py:110-111: uniform fallback
        const int64_t ii = rng.index(n);
        MG_CUDA(cudaMemcpyAsync(sel.p, &ii, sizeof(int64_t), cudaMemcpyHostToDevice, st));
      } else {
        const double rr = rng.uniform() * total;
        k_km_search<<<1, 32, 0, st>>>(n, cum.p, rr, sel.p);
        MG_CHECK_LAUNCH(ctx);
      }
      k_km_gather_row<<<1, 32, 0, st>>>(d, X, sel.p, C.p + (size_t)j * d);
      MG_CHECK_LAUNCH(ctx);
      k_km_d2<<<g, kKmThreads, 0, st>>>(n, d, X, C.p + (size_t)j * d, d2.p, 1);
      MG_CHECK_LAUNCH(ctx);
    }
    // ---- Lloyd (clustering.py:70-96)
    MG_CUDA(cudaMemsetAsync(lab.p, 0xff, n * sizeof(int64_t), st));  // labels = -1
    int64_t *cur = lab.p, *nxt = lab2.p;
    for (int it = 0; it < kKmMaxIter; ++it) {
      MG_CUDA(cudaMemsetAsync(counts.p, 0, c * sizeof(int), st));
      MG_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int), st));
      k_km_assign<<<g, kKmThreads, 0, st>>>(n, d, c, X, C.p, cur, nxt, fit.p, counts.p, changed.p);
      MG_CHECK_LAUNCH(ctx);
      std::vector<int> hc(c + 1);
      d2h_sync(ctx, hc.data(), counts.p, c * sizeof(int));
      bool repaired = false;
      for (int j = 0; j < c; ++j) {
        if (hc[j] != 0) continue;
        // steal the worst-fit point among clusters with > 1 member
        k_km_mask_fit<<<g, kKmThreads, 0, st>>>(n, nxt, fit.p, counts.p, d2.p);
        MG_CHECK_LAUNCH(ctx);
        size_t tb = tmp.n;
        MG_CUDA(cub::DeviceReduce::Reduce(tmp.p, tb, cub::ArgIndexInputIterator<const double *, int64_t>(d2.p),
                                          amax.p, n, ArgMax(),
                                          cub::KeyValuePair<int64_t, double>(0, -INFINITY), st));
        k_km_set_label<<<1, 32, 0, st>>>(nxt, reinterpret_cast<int64_t *>(amax.p), j, counts.p, n);
        MG_CHECK_LAUNCH(ctx);
        d2h_sync(ctx, hc.data(), counts.p, c * sizeof(int));
        repaired = true;
      }
      if (repaired) {  // compare the repaired labels (clustering.py:80)
        MG_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int), st));
        k_km_diff<<<g, kKmThreads, 0, st>>>(n, cur, nxt, changed.p);
        MG_CHECK_LAUNCH(ctx);
      }
      int ch;
      d2h_sync(ctx, &ch, changed.p, sizeof(int));
      if (!ch && it > 0) break;  // labels repeat (the initial -1 labels never do)
      std::swap(cur, nxt);
      k_km_sums<<<kKmBlocks, kKmThreads, 0, st>>>(n, d, c, X, cur, part.p);
      MG_CHECK_LAUNCH(ctx);
      k_km_centers<<<grid_for(c * d, 256, 64), 256, 0, st>>>(kKmBlocks, d, c, part.p, counts.p, C.p);
      MG_CHECK_LAUNCH(ctx);
    }
    // cur holds the final labels (nxt equals cur when converged)
    k_km_wcss<<<kKmBlocks, kKmThreads, 0, st>>>(n, d, X, C.p, cur, wpart.p);
    MG_CHECK_LAUNCH(ctx);
    std::vector<double> hw(kKmBlocks);
    d2h_sync(ctx, hw.data(), wpart.p, kKmBlocks * sizeof(double));
    double wcss = 0.0;
    for (double v : hw) wcss += v;
    if (r == 0 || wcss < best_wcss) {
      best_wcss = wcss;
      MG_CUDA(cudaMemcpyAsync(labels_out, cur, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
  }
  sync(ctx);
  return best_wcss;
}

}  // namespace mg
