// Row / disc queries of SparseSymMatrix and Graph (sparse.py:61-98,
// graph.py:93-96), balance_radii (operators.py:189-202), and numpy's pairwise
// summation on the device.
//
// np_sum_f64 reproduces numpy's DOUBLE_pairwise_sum bit for bit (the
// reduction behind np.sum / np.mean of a contiguous float64 array): blocks of
// <= 128 summed with 8 interleaved accumulators, larger ranges split at
// n/2 rounded down to a multiple of 8.  The recursion tree depends only on n,
// so it is cut at depth kPwDepth: 2^kPwDepth threads each sum one subtree
// (sequentially, in numpy's order), and one thread re-walks the top of the
// tree combining the subtree sums in the same order.
#include "mg_graph.cuh"

namespace mg {

namespace {

constexpr int kPwDepth = 12;

__device__ double pw_leaf(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
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

// numpy's split tree walked without recursion (post-order, explicit stack):
// leaf(off, len, depth, path) is summed for every node with len <= 128 or
// depth == max_depth, and sibling sums are added left + right
template <typename Leaf>
__device__ double pw_tree(int64_t n, int max_depth, Leaf leaf) {
  struct Fr {
    int64_t off, len;
    int depth;
    uint32_t path;
    int state;
    double left;
  };
  Fr st[64];
  int sp = 0;
  st[0] = {0, n, 0, 0u, 0, 0.0};
  double ret = 0.0;
  while (true) {
    Fr &f = st[sp];
    if (f.len <= 128 || f.depth == max_depth) {
      ret = leaf(f.off, f.len, f.depth, f.path);
    } else {
      int64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[sp + 1] = {f.off, n2, f.depth + 1, f.path * 2u, 0, 0.0};
        ++sp;
        continue;
      }
      if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[sp + 1] = {f.off + n2, f.len - n2, f.depth + 1, f.path * 2u + 1u, 0, 0.0};
        ++sp;
        continue;
      }
      ret = __dadd_rn(f.left, ret);
    }
    if (sp == 0) return ret;
    --sp;
  }
}

__device__ double pw_seq(const double *a, int64_t n) {
  return pw_tree(n, 64, [a](int64_t off, int64_t len, int, uint32_t) { return pw_leaf(a + off, len); });
}

// thread t: follow the bits of t (MSB first) for kPwDepth levels
__global__ void k_pw_subtrees(const double *__restrict__ a, int64_t n, double *__restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (1u << kPwDepth)) return;
  int64_t off = 0, len = n;
  for (int d = 0; d < kPwDepth; ++d) {
    if (len <= 128) {
      // leaf above the cut: owned by the thread whose remaining bits are 0
      if ((t & ((1u << (kPwDepth - d)) - 1)) != 0) return;
      break;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> (kPwDepth - 1 - d)) & 1u) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  out[t] = pw_seq(a + off, len);
}

__global__ void k_pw_top(int64_t n, const double *__restrict__ sub, double *__restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *out = n > 0 ? pw_tree(n, kPwDepth,
                         [sub](int64_t, int64_t, int d, uint32_t path) {
                           return sub[path << (kPwDepth - d)];
                         })
               : 0.0;
}

__global__ void k_sq(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dmul_rn(x[i], x[i]);
}

// sequential per-row sums in stored order (np.bincount(rows, weights=...))
__global__ void k_row_sums(int64_t n, const int64_t *__restrict__ ptr, const double *__restrict__ v,
                           double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) s = __dadd_rn(s, v[k]);
    out[i] = s;
  }
}

// gershgorin (sparse.py:84-94): center = stored diagonal (0 if absent), radius
// = sequential sum of |a_ij| over j != i; left = center - radius
__global__ void k_discs(int64_t n, const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                        const double *__restrict__ v, double *__restrict__ center,
                        double *__restrict__ radius, double *__restrict__ left) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double r = 0.0, d = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      if (idx[k] == i) {
        d = v[k];
        r = __dadd_rn(r, 0.0);  // the reference zeroes the diagonal entry, then sums
      } else {
        r = __dadd_rn(r, fabs(v[k]));
      }
    }
    if (center) center[i] = d;
    if (radius) radius[i] = r;
    if (left) left[i] = __dsub_rn(d, r);
  }
}

__global__ void k_log_all(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = log(x[i]);
}
__global__ void k_sub_all(double *__restrict__ y, const double *__restrict__ x, double c,
                          int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dsub_rn(x[i], c);
}
__global__ void k_scatter_perm(const double *__restrict__ x, const int64_t *__restrict__ perm,
                               double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[perm[i]] = x[i];
}
__global__ void k_exp_all(double *__restrict__ y, const double *__restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = exp(x[i]);
}

}  // namespace

double np_sum_f64(mg_ctx *ctx, const double *x, int64_t n) {
  if (n <= 0) return 0.0;
  DBuf<double> sub(ctx, ((size_t)1 << kPwDepth) + 1);
  k_pw_subtrees<<<(1 << kPwDepth) / 128, 128, 0, ctx->stream>>>(x, n, sub.p);
  MG_CHECK_LAUNCH(ctx);
  k_pw_top<<<1, 1, 0, ctx->stream>>>(n, sub.p, sub.p + (1 << kPwDepth));
  MG_CHECK_LAUNCH(ctx);
  double r;
  d2h_sync(ctx, &r, sub.p + (1 << kPwDepth), sizeof(double));
  return r;
}

double frobenius_np(mg_ctx *ctx, const double *data, int64_t nnz) {
  if (nnz <= 0) return 0.0;
  DBuf<double> sq(ctx, nnz);
  k_sq<<<grid_for(nnz, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(data, sq.p, nnz);
  MG_CHECK_LAUNCH(ctx);
  return std::sqrt(np_sum_f64(ctx, sq.p, nnz));
}

void row_sums(mg_ctx *ctx, int64_t n, const int64_t *ptr, const double *v, double *out) {
  if (n <= 0) return;
  k_row_sums<<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(n, ptr, v, out);
  MG_CHECK_LAUNCH(ctx);
}

void gershgorin(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *v,
                double *center, double *radius, double *left) {
  if (n <= 0) return;
  k_discs<<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(n, ptr, idx, v, center,
                                                                        radius, left);
  MG_CHECK_LAUNCH(ctx);
}

// operators.py:189-202: logb = log r - mean(log r); logb -= mean(logb); b = exp(logb);
// generalized_degree = exp(mean(log r)), means as numpy's pairwise sums / n
// With `perm` (row r is original node perm[r]) the means are taken over the
// original node order, as the reference sums them.
void balance_radii(mg_ctx *ctx, int64_t n, const double *radii, double *b, double *gdeg,
                   const int64_t *perm) {
  if (n <= 0) {
    *gdeg = NAN;
    return;
  }
  DBuf<double> logr(ctx, n), tmp(ctx, perm ? n : 1);
  const int g = grid_for(n, 256, ctx->num_sms * 16);
  auto mean = [&](const double *x) {
    if (!perm) return np_sum_f64(ctx, x, n) / (double)n;
    k_scatter_perm<<<g, 256, 0, ctx->stream>>>(x, perm, tmp.p, n);
    MG_CHECK_LAUNCH(ctx);
    return np_sum_f64(ctx, tmp.p, n) / (double)n;
  };
  k_log_all<<<g, 256, 0, ctx->stream>>>(radii, logr.p, n);
  MG_CHECK_LAUNCH(ctx);
  const double mean1 = mean(logr.p);
  k_sub_all<<<g, 256, 0, ctx->stream>>>(b, logr.p, mean1, n);  // b <- logb
  MG_CHECK_LAUNCH(ctx);
  const double mean2 = mean(b);
  k_sub_all<<<g, 256, 0, ctx->stream>>>(b, b, mean2, n);
  MG_CHECK_LAUNCH(ctx);
  k_exp_all<<<g, 256, 0, ctx->stream>>>(b, b, n);
  MG_CHECK_LAUNCH(ctx);
  *gdeg = exp(mean1);
}

}  // namespace mg
