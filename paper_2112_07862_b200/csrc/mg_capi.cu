// C ABI (include/manigraph_b200.h) + the end-to-end orchestration of
// identity_shift (operators.py:138-156 / eigensolver.py:431-460) and embed
// (embedding.py:77-103).  All exceptions are caught here and mapped to
// mg_status codes + a thread-local message.
#include <chrono>
#include <cmath>

#include "mg_block.cuh"
#include "mg_comm.cuh"
#include "mg_dist.cuh"
#include "mg_tc.cuh"
#include "mg_kmeans.cuh"
#include "mg_knn.cuh"
#include "mg_io.cuh"
#include "mg_rng.cuh"
#include "mg_graph.cuh"
#include "mg_small.cuh"

namespace mg {
const char *last_error_cstr();

// ---------------------------------------------------------- small helpers ---
__global__ void k_fill(double *x, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

__global__ void k_sq(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * x[i];
}

__global__ void k_diag_of(int64_t n, const int64_t *__restrict__ ptr,
                          const int64_t *__restrict__ idx, const double *__restrict__ data,
                          double *__restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
      if (idx[k] == i) v = data[k];
    d[i] = v;
  }
}

// densify a CSR (n <= 512) into row-major n x n
__global__ void k_densify(int64_t n, const int64_t *__restrict__ ptr,
                          const int64_t *__restrict__ idx, const double *__restrict__ data,
                          double *__restrict__ D) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t k = ptr[i] + threadIdx.x; k < ptr[i + 1]; k += blockDim.x)
      D[i * n + idx[k]] = data[k];
}

__global__ void __launch_bounds__(1024) k_dense_eigvals(double *D, int n, double *w_out) {
  __shared__ double cs[2 * 260];
  __shared__ int pidx[2 * 260];
  __shared__ int perm[512];
  __shared__ double w[512];
  __shared__ double red[1024];
  __shared__ int cnt;
  blk_jacobi(D, n, n, nullptr, 0, w, cs, pidx, perm, &cnt, red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) w_out[i] = w[i];
}

void dense_eigvals(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                   const double *data, double *w_host) {
  require(n <= 512, MG_ERR_INTERNAL, "dense eigensolve limited to n <= 512");
  DBuf<double> D(ctx, n * n), w(ctx, n);
  D.zero();
  k_densify<<<grid_for(n, 1, 65535), 128, 0, ctx->stream>>>(n, ptr, idx, data, D.p);
  MG_CHECK_LAUNCH(ctx);
  k_dense_eigvals<<<1, 1024, 0, ctx->stream>>>(D.p, (int)n, w.p);
  MG_CHECK_LAUNCH(ctx);
  d2h_sync(ctx, w_host, w.p, n * sizeof(double));
}

// ||A||_F as the reference computes it (sparse.py:76-77: numpy pairwise sum)
static double frobenius(mg_ctx *ctx, const double *data, int64_t nnz) {
  return frobenius_np(ctx, data, nnz);
}

static int64_t nnz_of(mg_ctx *ctx, const int64_t *ptr, int64_t n) {
  int64_t v = 0;
  d2h_sync(ctx, &v, ptr + n, sizeof(int64_t));
  return v;
}

// ------------------------------------------------------------- solver glue ---
struct SolverIn {
  int64_t n;
  const int64_t *ptr;
  const int64_t *idx;
  const double *data;
  int64_t nnz;
};

static SolveResult run_lobpcg(mg_ctx *ctx, const SolverIn &a, const double *b,
                              const mg_solver_cfg &cfg, const double *normals, int64_t n_normals,
                              const double *deflate, double *eigvecs,
                              const int64_t *perm = nullptr, Comm *comm = nullptr,
                              int n_deflate = 1) {
  SolveSpec sp;
  sp.perm = perm;
  sp.k = cfg.k;
  sp.max_iter = cfg.max_iter;
  sp.tol = cfg.tol;
  sp.jacobi = cfg.preconditioner != 0;
  sp.normals = normals;
  sp.n_normals = n_normals;
  sp.deflate = deflate;
  sp.n_deflate = deflate ? n_deflate : 0;
  sp.deflate_ld = a.n;  // column-major n x n_deflate (global n in the distributed mode)
  require(cfg.k >= 1, MG_ERR_INPUT, "block size must be >= 1, got " + std::to_string(cfg.k));
  require(cfg.tol > 0, MG_ERR_INPUT, "tolerance must be positive, got " + std::to_string(cfg.tol));
  require(cfg.k <= a.n, MG_ERR_INPUT,
          "block size " + std::to_string(cfg.k) + " exceeds dimension " + std::to_string(a.n));
  double anorm = frobenius(ctx, a.data, a.nnz) / std::sqrt((double)a.n);
  DBuf<double> diag(ctx, a.n);
  k_diag_of<<<grid_for(a.n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(a.n, a.ptr, a.idx,
                                                                            a.data, diag.p);
  MG_CHECK_LAUNCH(ctx);
  if (comm && comm->nranks > 1) {
    // 1-D row partition: the (replicated) matrix is cut into this rank's
    // rows with halo columns; b, diag and the deflation vector are sliced
    require(a.n < INT32_MAX, MG_ERR_INPUT, "distributed solve limited to n < 2^31");
    require(a.n >= 4 * (int64_t)comm->nranks, MG_ERR_INPUT,
            "distributed solve needs at least 4 rows per rank");
    sp.comm = comm;
    sp.n_global = a.n;
    if (cfg.precision == 1) {
      DistPart<float> dp;
      build_dist<float>(ctx, comm, a.n, a.ptr, a.idx, a.data, dp);
      sp.dist = &dp;
      sp.row_base = dp.r0;
      if (deflate) sp.deflate = deflate + dp.r0;
      return lobpcg<float>(ctx, dp.A.view, anorm, b + dp.r0, diag.p + dp.r0, sp, eigvecs);
    }
    DistPart<double> dp;
    build_dist<double>(ctx, comm, a.n, a.ptr, a.idx, a.data, dp);
    sp.dist = &dp;
    sp.row_base = dp.r0;
    if (deflate) sp.deflate = deflate + dp.r0;
    return lobpcg<double>(ctx, dp.A.view, anorm, b + dp.r0, diag.p + dp.r0, sp, eigvecs);
  }
  if (cfg.precision == 1) {
    OwnedCSR<float> A;
    make_solver_csr<float>(ctx, a.n, a.ptr, a.idx, a.data, A, a.nnz);
    return lobpcg<float>(ctx, A.view, anorm, b, diag.p, sp, eigvecs);
  }
  OwnedCSR<double> A;
  make_solver_csr<double>(ctx, a.n, a.ptr, a.idx, a.data, A, a.nnz);
  return lobpcg<double>(ctx, A.view, anorm, b, diag.p, sp, eigvecs);
}

static void check_b(mg_ctx *ctx, const double *b, int64_t n) {
  std::vector<double> hb(n);
  d2h_sync(ctx, hb.data(), b, n * sizeof(double));
  for (double v : hb)
    require(v > 0.0 && std::isfinite(v), MG_ERR_INPUT,
            "diagonal entries must be strictly positive and finite");
}

// smallest_above_null (eigensolver.py:431-460)
static double smallest_above_null_impl(mg_ctx *ctx, const SolverIn &q, double tau, double tol,
                                       int max_iter, const double *normals, int64_t n_normals,
                                       int precision, int *iters_out,
                                       const int64_t *perm = nullptr, Comm *comm = nullptr) {
  const int64_t n = q.n;
  if (n <= 512) {
    std::vector<double> w(n);
    dense_eigvals(ctx, n, q.ptr, q.idx, q.data, w.data());
    for (double v : w)
      if (v > tau) return v;
    return 0.0;
  }
  DBuf<double> ones(ctx, n), cvec(ctx, n);
  int g = grid_for(n, 256, ctx->num_sms * 16);
  k_fill<<<g, 256, 0, ctx->stream>>>(ones.p, n, 1.0);
  MG_CHECK_LAUNCH(ctx);
  k_fill<<<g, 256, 0, ctx->stream>>>(cvec.p, n, 1.0 / std::sqrt((double)n));
  MG_CHECK_LAUNCH(ctx);
  int k = 8;
  while (true) {
    mg_solver_cfg cfg{};
    cfg.k = (int)std::min<int64_t>(k, n - 1);
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    cfg.preconditioner = 1;
    cfg.precision = precision;
    DBuf<double> vecs(ctx, n * cfg.k);
    SolveResult r =
        run_lobpcg(ctx, q, ones.p, cfg, normals, n_normals, cvec.p, vecs.p, perm, comm);
    if (iters_out) *iters_out += r.iterations;
    for (double v : r.eigenvalues)
      if (v > tau) return v;
    if (k >= std::min<int64_t>(64, n - 1)) return 0.0;
    k *= 2;
  }
}

// identity_shift (operators.py:138-156)
static double identity_shift_impl(mg_ctx *ctx, const SolverIn &q, const double *normals,
                                  int64_t n_normals, int precision, int *iters_out,
                                  const int64_t *perm = nullptr, Comm *comm = nullptr) {
  if (iters_out) *iters_out = 0;
  require(check_symmetric(ctx, q.n, q.ptr, q.idx, q.data, 1e-12), MG_ERR_INPUT,
          "matrix is not symmetric");
  const int64_t n = q.n;
  if (n == 0 || q.nnz == 0) return 0.0;
  double tau = 1e-8 * trace(ctx, n, q.ptr, q.idx, q.data) / (double)n;
  return smallest_above_null_impl(ctx, q, tau, 1e-6, 60, normals, n_normals, precision, iters_out,
                                  perm, comm);
}

__global__ void k_scatter_rows(int64_t n, const double *__restrict__ src,
                               const int64_t *__restrict__ perm, double *__restrict__ dst) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[perm[r]] = src[r];
}

__global__ void k_drop_first_col(int64_t n, int K, const double *__restrict__ src,
                                 double *__restrict__ dst) {
  int64_t total = n * (int64_t)K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / K;
    int c = (int)(e - r * K);
    dst[e] = src[r * (K + 1) + c + 1];
  }
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void fill_out(const SolveResult &r, mg_solver_out *out, int k) {
  if (!out) return;
  for (int j = 0; j < k; ++j) {
    if (out->eigenvalues) out->eigenvalues[j] = r.eigenvalues[j];
    if (out->residual_norms) out->residual_norms[j] = r.residual_norms[j];
    if (out->converged) out->converged[j] = r.converged[j];
  }
  out->iterations = r.iterations;
  out->history_len = (int32_t)r.history.size();
  if (out->history)
    for (int i = 0; i < (int)r.history.size() && i < out->history_cap; ++i)
      out->history[i] = r.history[i];
  out->normals_used = (int32_t)std::min<int64_t>(r.normals_used, INT32_MAX);
}

// embed (embedding.py:77-103) on device arrays
static int embed_impl(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                      const double *w, int32_t K, const mg_solver_cfg *cfg_in, int literal,
                      int require_conv, int check_conn, const double *normals, int64_t n_normals,
                      double *P, double *b_out, mg_solver_out *out, mg_embed_diag *diag,
                      Comm *comm = nullptr) {
  double t0 = now_s();
  mg_embed_diag d{};
  require(K >= 1 && K <= n - 1, MG_ERR_INPUT,
          "embedding dimension must be in [1, " + std::to_string(n - 1) +
              "] (one extra eigenpair is solved and discarded), got " + std::to_string(K));
  mg_solver_cfg cfg = *cfg_in;
  cfg.k = K + 1;
  require(cfg.tol > 0, MG_ERR_INPUT, "tolerance must be positive, got " + std::to_string(cfg.tol));
  d.n_components = 1;
  if (check_conn) {
    int64_t count = components(ctx, n, ptr, idx, nullptr);
    d.n_components = count;
    if (count != 1) {
      if (diag) *diag = d;
      throw Error(MG_ERR_DISCONNECTED, "graph has " + std::to_string(count) +
                                           " connected components; embed the largest one");
    }
  }
  int64_t gnnz = nnz_of(ctx, ptr, n);
  // locality order for the solver: relabel the graph once, map results back
  DBuf<int64_t> perm, inv, pptr, pidx;
  DBuf<double> pw;
  const int64_t *perm_p = nullptr;
  if (cfg.reorder && n > 4096) {
    perm.alloc(ctx, n);
    inv.alloc(ctx, n);
    cm_order(ctx, n, ptr, idx, perm.p, inv.p);
    pptr.alloc(ctx, n + 1);
    pidx.alloc(ctx, gnnz > 0 ? gnnz : 1);
    pw.alloc(ctx, gnnz > 0 ? gnnz : 1);
    permute_graph(ctx, n, ptr, idx, w, perm.p, inv.p, pptr.p, pidx.p, pw.p);
    ptr = pptr.p;
    idx = pidx.p;
    w = pw.p;
    perm_p = perm.p;
  }
  // L (graph.py:321-346)
  DBuf<int64_t> lptr(ctx, n + 1), lidx(ctx, gnnz + n);
  DBuf<double> ldata(ctx, gnnz + n);
  laplacian(ctx, n, ptr, idx, w, lptr.p, lidx.p, ldata.p);
  // T, Q (operators.py:88-135)
  DBuf<int64_t> tptr(ctx, n + 1);
  int64_t tnnz = two_hop_count(ctx, n, ptr, idx, tptr.p);
  DBuf<int64_t> tidx(ctx, tnnz > 0 ? tnnz : 1);
  two_hop_fill(ctx, n, ptr, idx, tptr.p, tidx.p);
  DBuf<int64_t> qptr(ctx, n + 1);
  int64_t qnnz = q_count(ctx, n, tptr.p, qptr.p);
  DBuf<int64_t> qidx(ctx, qnnz > 0 ? qnnz : 1);
  DBuf<double> qdata(ctx, qnnz > 0 ? qnnz : 1);
  q_fill(ctx, n, tptr.p, tidx.p, literal, qptr.p, qidx.p, qdata.p);
  tidx.release();
  d.t_nnz = tnnz;
  d.q_nnz = qnnz;
  double t1 = now_s();
  // eps (operators.py:138-156)
  SolverIn qin{n, qptr.p, qidx.p, qdata.p, qnnz};
  int eps_it = 0;
  double eps =
      identity_shift_impl(ctx, qin, normals, n_normals, cfg.precision, &eps_it, perm_p, comm);
  double t2 = now_s();
  double mu = repulsion_weight(ctx, n, qptr.p, qidx.p, qdata.p, eps);
  DBuf<int64_t> aptr(ctx, n + 1);
  int64_t annz = assemble_count(ctx, n, lptr.p, lidx.p, ldata.p, qptr.p, qidx.p, qdata.p, mu, eps,
                                aptr.p);
  DBuf<int64_t> aidx(ctx, annz > 0 ? annz : 1);
  DBuf<double> adata(ctx, annz > 0 ? annz : 1);
  assemble_fill(ctx, n, lptr.p, lidx.p, ldata.p, qptr.p, qidx.p, qdata.p, mu, eps, aptr.p, aidx.p,
                adata.p);
  lidx.release();
  ldata.release();
  qidx.release();
  qdata.release();
  double gdeg = 0;
  DBuf<double> bperm;
  double *b_solver = b_out;
  if (perm_p) {
    bperm.alloc(ctx, n);
    b_solver = bperm.p;
  }
  int64_t bad = degree_balancing(ctx, n, aptr.p, aidx.p, adata.p, b_solver, &gdeg, perm_p);
  if (bad >= 0)
    throw Error(MG_ERR_DISCONNECTED, "node " + std::to_string(bad) +
                                         " has no off-diagonal coupling; extract the largest "
                                         "connected component and retry");
  double minleft;
  int64_t brow;
  disc_left_min(ctx, n, aptr.p, aidx.p, adata.p, &minleft, &brow, perm_p);
  if (perm_p) {  // b in the caller's node order
    k_scatter_rows<<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(n, b_solver,
                                                                                perm_p, b_out);
    MG_CHECK_LAUNCH(ctx);
  }
  d.mu = mu;
  d.epsilon = eps;
  d.min_disc_left_end = minleft;
  d.binding_row = brow;
  d.a_nnz = annz;
  d.generalized_degree = gdeg;
  d.eps_iterations = eps_it;
  double t3 = now_s();
  // solve K+1 pairs and drop the first (embedding.py:61-74, 94-103)
  DBuf<double> vecs(ctx, n * (int64_t)cfg.k);
  SolverIn ain{n, aptr.p, aidx.p, adata.p, annz};
  SolveResult r =
      run_lobpcg(ctx, ain, b_solver, cfg, normals, n_normals, nullptr, vecs.p, perm_p, comm);
  const bool full = cfg_in->reserved == 1;  // caller wants all K+1 pairs (drop done by caller)
  if (full) {
    MG_CUDA(cudaMemcpyAsync(P, vecs.p, n * (int64_t)cfg.k * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    k_drop_first_col<<<grid_for(n * K, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(n, K,
                                                                                       vecs.p, P);
    MG_CHECK_LAUNCH(ctx);
  }
  sync(ctx);
  double t4 = now_s();
  d.iterations = r.iterations;
  d.fast_steps = r.fast_steps;
  d.fast_fallbacks = r.fast_fallbacks;
  d.dropped_eigenvalue = r.eigenvalues[0];
  d.seconds_setup = (t1 - t0) + (t3 - t2);
  d.seconds_eps = t2 - t1;
  d.seconds_solve = t4 - t3;
  if (out) {
    SolveResult rr = r;
    rr.eigenvalues.erase(rr.eigenvalues.begin());
    // residuals / converged keep all K+1 pairs (diagnostics carry the solver's view)
    for (int j = 0; j < (full ? K + 1 : K); ++j) {
      if (out->eigenvalues) out->eigenvalues[j] = r.eigenvalues[full ? j : j + 1];
    }
    for (int j = 0; j < K + 1; ++j) {
      if (out->residual_norms) out->residual_norms[j] = r.residual_norms[j];
      if (out->converged) out->converged[j] = r.converged[j];
    }
    out->iterations = r.iterations;
    out->history_len = (int32_t)r.history.size();
    if (out->history)
      for (int i = 0; i < (int)r.history.size() && i < out->history_cap; ++i)
        out->history[i] = r.history[i];
    out->normals_used = (int32_t)std::min<int64_t>(r.normals_used, INT32_MAX);
  }
  if (diag) *diag = d;
  if (require_conv) {
    int bad_pairs = 0;
    for (int c : r.converged) bad_pairs += c ? 0 : 1;
    if (bad_pairs)
      throw Error(MG_ERR_NOT_CONVERGED,
                  "embedding eigensolve: " + std::to_string(bad_pairs) + " of " +
                      std::to_string(cfg.k) + " eigenpairs unconverged after " +
                      std::to_string(r.iterations) + " iterations");
  }
  return MG_OK;
}

}  // namespace mg

using namespace mg;

#define MG_API_BEGIN(ctx)                                           \
  try {                                                             \
    if (ctx) MG_CUDA(cudaSetDevice((ctx)->device));
#define MG_API_END                                                  \
  return MG_OK;                                                     \
  }                                                                 \
  catch (const mg::Error &e) {                                      \
    mg::set_last_error(e.what());                                   \
    return e.code;                                                  \
  }                                                                 \
  catch (const std::exception &e) {                                 \
    mg::set_last_error(e.what());                                   \
    return MG_ERR_INTERNAL;                                         \
  }

extern "C" {

int mg_version(void) { return 1; }
const char *mg_last_error(void) { return mg::last_error_cstr(); }

int mg_device_count(int *count) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  MG_CUDA(cudaGetDeviceCount(count));
  MG_API_END
}

int mg_ctx_create(int device, void *stream, mg_ctx **out) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  MG_CUDA(cudaSetDevice(device));
  mg_ctx *c = new mg_ctx();
  c->device = device;
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    MG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  int sms = 0;
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  c->num_sms = sms;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  MG_API_END
}

int mg_ctx_destroy(mg_ctx *ctx) {
  MG_API_BEGIN(ctx)
  if (!ctx) return MG_OK;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  free_stages(ctx);
  for (auto &r : ctx->prof) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  delete ctx;
  MG_API_END
}

int mg_ctx_set_stream(mg_ctx *ctx, void *stream) {
  MG_API_BEGIN(ctx)
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
  } else {
    MG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  MG_API_END
}

int mg_ctx_launch_count(mg_ctx *ctx, int64_t *count) {
  MG_API_BEGIN(ctx)
  *count = ctx->launches;
  MG_API_END
}

int mg_ctx_get_stream(mg_ctx *ctx, void **stream) {
  MG_API_BEGIN(ctx)
  *stream = (void *)ctx->stream;
  MG_API_END
}

int mg_ctx_set_profiling(mg_ctx *ctx, int enable) {
  MG_API_BEGIN(ctx)
  ctx->profiling = enable;
  MG_API_END
}

int mg_ctx_stats(mg_ctx *ctx, int64_t *counts, double *milliseconds, double *bytes) {
  MG_API_BEGIN(ctx)
  sync(ctx);
  for (int c = 0; c < PROF_NCLASS; ++c) {
    counts[c] = 0;
    milliseconds[c] = 0.0;
    bytes[c] = 0.0;
  }
  for (auto &r : ctx->prof) {
    float ms = 0.f;
    MG_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
    counts[r.cls] += 1;
    milliseconds[r.cls] += ms;
    bytes[r.cls] += r.bytes;
    ctx->event_pool.push_back(r.start);
    ctx->event_pool.push_back(r.stop);
  }
  ctx->prof.clear();
  MG_API_END
}

int mg_components(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  int64_t *labels, int64_t *count) {
  MG_API_BEGIN(ctx)
  *count = components(ctx, n, indptr, indices, labels);
  sync(ctx);
  MG_API_END
}

int mg_laplacian(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                 const double *weights, int64_t *out_indptr, int64_t *out_indices,
                 double *out_data) {
  MG_API_BEGIN(ctx)
  laplacian(ctx, n, indptr, indices, weights, out_indptr, out_indices, out_data);
  sync(ctx);
  MG_API_END
}

int mg_two_hop_count(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                     int64_t *t_indptr, int64_t *t_nnz) {
  MG_API_BEGIN(ctx)
  *t_nnz = two_hop_count(ctx, n, indptr, indices, t_indptr);
  MG_API_END
}

int mg_two_hop_fill(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const int64_t *t_indptr, int64_t *t_indices) {
  MG_API_BEGIN(ctx)
  two_hop_fill(ctx, n, indptr, indices, t_indptr, t_indices);
  sync(ctx);
  MG_API_END
}

int mg_two_hop_laplacian_count(mg_ctx *ctx, int64_t n, const int64_t *t_indptr,
                               int64_t *q_indptr, int64_t *q_nnz) {
  MG_API_BEGIN(ctx)
  *q_nnz = q_count(ctx, n, t_indptr, q_indptr);
  MG_API_END
}

int mg_two_hop_laplacian_fill(mg_ctx *ctx, int64_t n, const int64_t *t_indptr,
                              const int64_t *t_indices, int literal_diagonal,
                              const int64_t *q_indptr, int64_t *q_indices, double *q_data) {
  MG_API_BEGIN(ctx)
  q_fill(ctx, n, t_indptr, t_indices, literal_diagonal, q_indptr, q_indices, q_data);
  sync(ctx);
  MG_API_END
}

int mg_check_symmetric(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                       const double *data, double rtol, int *is_symmetric) {
  MG_API_BEGIN(ctx)
  *is_symmetric = check_symmetric(ctx, n, indptr, indices, data, rtol) ? 1 : 0;
  MG_API_END
}

int mg_repulsion_weight(mg_ctx *ctx, int64_t n, const int64_t *q_indptr,
                        const int64_t *q_indices, const double *q_data, double epsilon,
                        double *mu) {
  MG_API_BEGIN(ctx)
  *mu = repulsion_weight(ctx, n, q_indptr, q_indices, q_data, epsilon);
  MG_API_END
}

int mg_assemble_count(mg_ctx *ctx, int64_t n, const int64_t *l_indptr, const int64_t *l_indices,
                      const double *l_data, const int64_t *q_indptr, const int64_t *q_indices,
                      const double *q_data, double mu, double epsilon, int64_t *a_indptr,
                      int64_t *a_nnz) {
  MG_API_BEGIN(ctx)
  *a_nnz = assemble_count(ctx, n, l_indptr, l_indices, l_data, q_indptr, q_indices, q_data, mu,
                          epsilon, a_indptr);
  MG_API_END
}

int mg_assemble_fill(mg_ctx *ctx, int64_t n, const int64_t *l_indptr, const int64_t *l_indices,
                     const double *l_data, const int64_t *q_indptr, const int64_t *q_indices,
                     const double *q_data, double mu, double epsilon, const int64_t *a_indptr,
                     int64_t *a_indices, double *a_data) {
  MG_API_BEGIN(ctx)
  assemble_fill(ctx, n, l_indptr, l_indices, l_data, q_indptr, q_indices, q_data, mu, epsilon,
                a_indptr, a_indices, a_data);
  sync(ctx);
  MG_API_END
}

int mg_degree_balancing(mg_ctx *ctx, int64_t n, const int64_t *a_indptr,
                        const int64_t *a_indices, const double *a_data, double *b,
                        double *generalized_degree, int64_t *isolated_node) {
  MG_API_BEGIN(ctx)
  int64_t bad = degree_balancing(ctx, n, a_indptr, a_indices, a_data, b, generalized_degree);
  sync(ctx);
  if (isolated_node) *isolated_node = bad;
  if (bad >= 0)
    throw Error(MG_ERR_DISCONNECTED, "node " + std::to_string(bad) +
                                         " has no off-diagonal coupling; extract the largest "
                                         "connected component and retry");
  MG_API_END
}

int mg_row_sums(mg_ctx *ctx, int64_t n, const int64_t *indptr, const double *data,
                double *out) {
  MG_API_BEGIN(ctx)
  require(n >= 0, MG_ERR_INPUT, "n must be non-negative");
  row_sums(ctx, n, indptr, data, out);
  sync(ctx);
  MG_API_END
}

int mg_gershgorin(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *data, double *centers, double *radii, double *left_ends) {
  MG_API_BEGIN(ctx)
  require(n >= 0, MG_ERR_INPUT, "n must be non-negative");
  gershgorin(ctx, n, indptr, indices, data, centers, radii, left_ends);
  sync(ctx);
  MG_API_END
}

int mg_frobenius_norm(mg_ctx *ctx, int64_t nnz, const double *data, double *out) {
  MG_API_BEGIN(ctx)
  require(nnz >= 0 && out != nullptr, MG_ERR_INPUT, "bad frobenius_norm arguments");
  *out = frobenius_np(ctx, data, nnz);
  MG_API_END
}

int mg_balance_radii(mg_ctx *ctx, int64_t n, const double *radii, double *b,
                     double *generalized_degree) {
  MG_API_BEGIN(ctx)
  require(n >= 0 && generalized_degree != nullptr, MG_ERR_INPUT, "bad balance_radii arguments");
  balance_radii(ctx, n, radii, b, generalized_degree);
  sync(ctx);
  MG_API_END
}

int mg_disc_left_min(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
                     const double *a_data, double *min_left, int64_t *binding_row) {
  MG_API_BEGIN(ctx)
  disc_left_min(ctx, n, a_indptr, a_indices, a_data, min_left, binding_row);
  MG_API_END
}

int mg_lobpcg(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
              const double *a_data, const double *b, const mg_solver_cfg *cfg,
              const double *normals, int64_t n_normals, const double *deflate,
              double *eigenvectors, mg_solver_out *out) {
  MG_API_BEGIN(ctx)
  require(cfg != nullptr, MG_ERR_INPUT, "cfg is NULL");
  check_b(ctx, b, n);
  SolverIn a{n, a_indptr, a_indices, a_data, nnz_of(ctx, a_indptr, n)};
  SolveResult r = run_lobpcg(ctx, a, b, *cfg, normals, n_normals, deflate, eigenvectors);
  fill_out(r, out, cfg->k);
  MG_API_END
}

int mg_lobpcg_deflate(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
                      const double *a_data, const double *b, const mg_solver_cfg *cfg,
                      const double *normals, int64_t n_normals, const double *deflate,
                      int32_t n_deflate, double *eigenvectors, mg_solver_out *out) {
  MG_API_BEGIN(ctx)
  require(cfg != nullptr, MG_ERR_INPUT, "cfg is NULL");
  require(n_deflate >= 0 && (n_deflate == 0 || deflate != nullptr), MG_ERR_INPUT,
          "deflate is NULL with n_deflate > 0");
  check_b(ctx, b, n);
  SolverIn a{n, a_indptr, a_indices, a_data, nnz_of(ctx, a_indptr, n)};
  SolveResult r = run_lobpcg(ctx, a, b, *cfg, normals, n_normals, n_deflate ? deflate : nullptr,
                             eigenvectors, nullptr, nullptr, n_deflate);
  fill_out(r, out, cfg->k);
  MG_API_END
}

int mg_identity_shift(mg_ctx *ctx, int64_t n, const int64_t *q_indptr, const int64_t *q_indices,
                      const double *q_data, const double *normals, int64_t n_normals,
                      int32_t precision, double *epsilon) {
  MG_API_BEGIN(ctx)
  SolverIn q{n, q_indptr, q_indices, q_data, nnz_of(ctx, q_indptr, n)};
  *epsilon = identity_shift_impl(ctx, q, normals, n_normals, precision, nullptr);
  MG_API_END
}

int mg_smallest_above_null(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                           const double *data, double tau, double tol, int32_t max_iter,
                           const double *normals, int64_t n_normals, int32_t precision,
                           double *value) {
  MG_API_BEGIN(ctx)
  SolverIn q{n, indptr, indices, data, nnz_of(ctx, indptr, n)};
  *value = smallest_above_null_impl(ctx, q, tau, tol, max_iter, normals, n_normals, precision,
                                    nullptr);
  MG_API_END
}

int mg_spmm(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
            const double *data, const double *X, int32_t k, double *Y) {
  MG_API_BEGIN(ctx)
  require(k >= 1, MG_ERR_INPUT, "block width must be >= 1");
  OwnedCSR<double> A;
  make_solver_csr<double>(ctx, n, indptr, indices, data, A, nnz_of(ctx, indptr, n));
  int kp = (k + 1) / 2 * 2;
  if (kp == k) {
    spmm<double>(ctx, A.view, X, k, Y, k, k);
  } else {  // pad to the 16-byte row granule
    DBuf<double> xp(ctx, n * kp), yp(ctx, n * kp);
    MG_CUDA(cudaMemcpy2DAsync(xp.p, kp * sizeof(double), X, k * sizeof(double),
                              k * sizeof(double), n, cudaMemcpyDeviceToDevice, ctx->stream));
    MG_CUDA(cudaMemset2DAsync(xp.p + k, kp * sizeof(double), 0, (kp - k) * sizeof(double), n,
                              ctx->stream));
    spmm<double>(ctx, A.view, xp.p, kp, yp.p, kp, kp);
    MG_CUDA(cudaMemcpy2DAsync(Y, k * sizeof(double), yp.p, kp * sizeof(double),
                              k * sizeof(double), n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  sync(ctx);
  MG_API_END
}

int mg_embed(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
             const double *weights, int32_t K, const mg_solver_cfg *cfg, int32_t literal_diagonal,
             int32_t require_convergence, int32_t check_connected, const double *normals,
             int64_t n_normals, double *P, double *b, mg_solver_out *out, mg_embed_diag *diag) {
  MG_API_BEGIN(ctx)
  require(cfg != nullptr, MG_ERR_INPUT, "cfg is NULL");
  return embed_impl(ctx, n, indptr, indices, weights, K, cfg, literal_diagonal,
                    require_convergence, check_connected, normals, n_normals, P, b, out, diag);
  MG_API_END
}

int mg_gram_pair_f32(mg_ctx *ctx, int64_t n, int32_t ld, int32_t w, const float *S,
                     const float *AS, const float *b, double *GB, double *GA) {
  MG_API_BEGIN(ctx)
  require(n >= 1 && w >= 1 && ld >= w, MG_ERR_INPUT, "bad Gram shape");
  require(gram_tc_supported(w), MG_ERR_INPUT,
          "tensor-core Gram pair needs 48 < w <= 128, w % 4 == 0 (and MG_TC != 0)");
  DBuf<double> part;
  gram_pair_tc(ctx, n, ld, w, S, AS, b, GB, GA, part);
  sync(ctx);
  MG_API_END
}

int mg_update_f32(mg_ctx *ctx, int32_t variant, int64_t n, int32_t ld, int32_t m, int32_t mp,
                  float *S, float *AS, const float *b, const float *prec, const float *M,
                  const double *theta, float *wc, double *colsums) {
  MG_API_BEGIN(ctx)
  require(n >= 1 && m >= 1 && mp >= m && mp % 4 == 0 && ld >= 3 * mp && ld % 4 == 0, MG_ERR_INPUT,
          "bad update shape");
  require(variant == 0 || update_tc3_supported(3 * mp, mp, ld), MG_ERR_INPUT,
          "tensor-core update needs 3 mp <= 128");
  update_f32_hook(ctx, variant, n, ld, m, mp, S, AS, b, prec, M, theta, wc, colsums);
  sync(ctx);
  MG_API_END
}

int mg_copy_d2h(mg_ctx *ctx, void *host, const void *dev, int64_t bytes) {
  MG_API_BEGIN(ctx)
  require(bytes >= 0 && (bytes == 0 || (host && dev)), MG_ERR_INPUT, "bad copy arguments");
  d2h_sync(ctx, host, dev, (size_t)bytes);
  MG_API_END
}

int mg_copy_h2d(mg_ctx *ctx, void *dev, const void *host, int64_t bytes) {
  MG_API_BEGIN(ctx)
  require(bytes >= 0 && (bytes == 0 || (host && dev)), MG_ERR_INPUT, "bad copy arguments");
  h2d(ctx, dev, host, (size_t)bytes);
  MG_API_END
}

int mg_normal_stream(mg_ctx *ctx, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, int64_t count, double *out) {
  MG_API_BEGIN(ctx)
  require(out != nullptr || count == 0, MG_ERR_INPUT, "out is NULL");
  normal_stream(ctx, state_hi, state_lo, inc_hi, inc_lo, count, out);
  MG_API_END
}

int mg_save_embedding_csv(const char *path, int64_t n, int32_t k, const double *P,
                          int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr, MG_ERR_INPUT, "path is NULL");
  save_embedding_csv(path, n, k, P, threads);
  MG_API_END
}

int mg_load_embedding_csv_dims(const char *path, int64_t *n, int32_t *k) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && n != nullptr && k != nullptr, MG_ERR_INPUT, "NULL argument");
  int kk = 0;
  load_embedding_csv(path, n, &kk, nullptr, 1);
  *k = kk;
  MG_API_END
}

int mg_load_embedding_csv(const char *path, int64_t n, int32_t k, double *P, int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && P != nullptr, MG_ERR_INPUT, "NULL argument");
  int64_t n2 = 0;
  int k2 = 0;
  load_embedding_csv(path, &n2, &k2, nullptr, 1);
  require(n2 == n && k2 == k, MG_ERR_INPUT, "embedding dimensions changed between calls");
  load_embedding_csv(path, &n2, &k2, P, threads);
  MG_API_END
}

int mg_save_edge_list(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                      const double *weights, int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && indptr != nullptr, MG_ERR_INPUT, "NULL argument");
  save_edge_list(path, n, indptr, indices, weights, threads);
  MG_API_END
}

static thread_local mg::EdgeListResult tl_edges;

int mg_load_edge_list_count(const char *path, int32_t threads, int64_t *n, int64_t *nnz,
                            int64_t *err_line) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && n != nullptr && nnz != nullptr, MG_ERR_INPUT, "NULL argument");
  tl_edges = mg::EdgeListResult();
  try {
    load_edge_list(path, threads, tl_edges);
  } catch (...) {
    if (err_line) *err_line = tl_edges.err_line;
    throw;
  }
  *n = tl_edges.n;
  *nnz = (int64_t)tl_edges.indices.size();
  MG_API_END
}

int mg_load_edge_list_fill(int64_t *indptr, int64_t *indices, double *weights) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(indptr != nullptr && !tl_edges.indptr.empty(), MG_ERR_INPUT,
          "mg_load_edge_list_fill without a successful mg_load_edge_list_count");
  std::memcpy(indptr, tl_edges.indptr.data(), tl_edges.indptr.size() * sizeof(int64_t));
  std::memcpy(indices, tl_edges.indices.data(), tl_edges.indices.size() * sizeof(int64_t));
  std::memcpy(weights, tl_edges.weights.data(), tl_edges.weights.size() * sizeof(double));
  tl_edges = mg::EdgeListResult();
  MG_API_END
}

int mg_save_embedding_bin(const char *path, int64_t n, int32_t k, const double *P,
                          const double *eigenvalues, const double *b, const char *method,
                          int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && (P != nullptr || n * (int64_t)k == 0), MG_ERR_INPUT, "NULL argument");
  save_embedding_bin(path, n, k, P, eigenvalues, b, method, threads);
  MG_API_END
}

int mg_load_embedding_bin_dims(const char *path, int64_t *n, int32_t *k, int32_t *has_b,
                               char *method16) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && n != nullptr && k != nullptr && has_b != nullptr, MG_ERR_INPUT,
          "NULL argument");
  int64_t kk = 0;
  int hb = 0;
  load_embedding_bin(path, n, &kk, &hb, method16, nullptr, nullptr, nullptr, 1);
  *k = (int32_t)kk;
  *has_b = hb;
  MG_API_END
}

int mg_load_embedding_bin(const char *path, double *P, double *eigenvalues, double *b,
                          int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && P != nullptr, MG_ERR_INPUT, "NULL argument");
  int64_t n = 0, k = 0;
  int hb = 0;
  load_embedding_bin(path, &n, &k, &hb, nullptr, P, eigenvalues, b, threads);
  MG_API_END
}

int mg_save_graph_bin(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                      const double *weights, int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && indptr != nullptr, MG_ERR_INPUT, "NULL argument");
  save_graph_bin(path, n, indptr, indices, weights, threads);
  MG_API_END
}

int mg_load_graph_bin_dims(const char *path, int64_t *n, int64_t *nnz) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && n != nullptr && nnz != nullptr, MG_ERR_INPUT, "NULL argument");
  load_graph_bin(path, n, nnz, nullptr, nullptr, nullptr, 1);
  MG_API_END
}

int mg_load_graph_bin(const char *path, int64_t *indptr, int64_t *indices, double *weights,
                      int32_t threads) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(path != nullptr && indptr != nullptr, MG_ERR_INPUT, "NULL argument");
  int64_t n = 0, nnz = 0;
  load_graph_bin(path, &n, &nnz, indptr, indices, weights, threads);
  MG_API_END
}

int mg_knn_graph_count(mg_ctx *ctx, int64_t n, int32_t d, const double *X, int32_t k,
                       int32_t weighted, int64_t *indptr, int64_t *nnz) {
  MG_API_BEGIN(ctx)
  require(X != nullptr && indptr != nullptr && nnz != nullptr, MG_ERR_INPUT, "NULL argument");
  KnnResult r = knn_graph(ctx, n, d, X, k, weighted != 0);
  MG_CUDA(cudaMemcpyAsync(indptr, r.indptr.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                          ctx->stream));
  *nnz = r.nnz;
  sync(ctx);
  MG_API_END
}

int mg_knn_graph_fill(mg_ctx *ctx, int64_t n, int32_t d, const double *X, int32_t k,
                      int32_t weighted, int64_t *indices, double *weights) {
  MG_API_BEGIN(ctx)
  require(X != nullptr && indices != nullptr && weights != nullptr, MG_ERR_INPUT, "NULL argument");
  KnnResult r = knn_graph(ctx, n, d, X, k, weighted != 0);
  if (r.nnz) {
    MG_CUDA(cudaMemcpyAsync(indices, r.indices.p, r.nnz * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    MG_CUDA(cudaMemcpyAsync(weights, r.weights.p, r.nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx->stream));
  }
  sync(ctx);
  MG_API_END
}

int mg_kmeans(mg_ctx *ctx, int64_t n, int32_t d, const double *points, int32_t c,
              int32_t restarts, uint64_t seed, int64_t *labels, double *wcss) {
  MG_API_BEGIN(ctx)
  require(points != nullptr && labels != nullptr, MG_ERR_INPUT, "points / labels is NULL");
  const double v = kmeans(ctx, n, d, points, c, restarts, seed, labels);
  if (wcss) *wcss = v;
  MG_API_END
}

int mg_normalize_rows(mg_ctx *ctx, int64_t n, int32_t d, const double *points, double *out) {
  MG_API_BEGIN(ctx)
  normalize_rows(ctx, n, d, points, out);
  sync(ctx);
  MG_API_END
}

int mg_nccl_unique_id(uint8_t *uid) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(uid != nullptr, MG_ERR_INPUT, "uid is NULL");
  nccl_unique_id(uid);
  MG_API_END
}

int mg_comm_create_nccl(mg_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *uid,
                        mg_comm **out) {
  MG_API_BEGIN(ctx)
  require(ctx && uid && out, MG_ERR_INPUT, "NULL argument");
  require(nranks >= 1 && rank >= 0 && rank < nranks, MG_ERR_INPUT, "bad rank / world size");
  auto *c = new mg_comm();
  try {
    c->impl = make_nccl_comm(nranks, rank, uid);
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  MG_API_END
}

int mg_local_group_create(int32_t nranks, void **group) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(nranks >= 1 && group, MG_ERR_INPUT, "bad arguments");
  *group = local_comm_group_create(nranks);
  MG_API_END
}

int mg_local_group_destroy(void *group) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  local_comm_group_destroy(group);
  MG_API_END
}

int mg_comm_create_local(void *group, int32_t rank, mg_comm **out) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(group && out, MG_ERR_INPUT, "NULL argument");
  auto *c = new mg_comm();
  c->impl = local_comm_rank(group, rank);
  *out = c;
  MG_API_END
}

int mg_comm_destroy(mg_comm *comm) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  if (comm) {
    delete comm->impl;
    delete comm;
  }
  MG_API_END
}

int mg_embed_dist(mg_ctx *ctx, mg_comm *comm, int64_t n, const int64_t *indptr,
                  const int64_t *indices, const double *weights, int32_t K,
                  const mg_solver_cfg *cfg, int32_t literal_diagonal, int32_t require_convergence,
                  int32_t check_connected, const double *normals, int64_t n_normals, double *P,
                  double *b, mg_solver_out *out, mg_embed_diag *diag) {
  MG_API_BEGIN(ctx)
  require(cfg != nullptr && comm != nullptr, MG_ERR_INPUT, "cfg / comm is NULL");
  return embed_impl(ctx, n, indptr, indices, weights, K, cfg, literal_diagonal,
                    require_convergence, check_connected, normals, n_normals, P, b, out, diag,
                    comm->impl);
  MG_API_END
}

int mg_dist_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, int32_t nranks,
                      int32_t rank, mg_dist_plan_info *info, int64_t *halo, int64_t *roff,
                      int64_t *rcnt, int64_t *soff, int64_t *scnt, int32_t *send_rows,
                      int32_t *local_indices) {
  MG_API_BEGIN((mg_ctx *)nullptr)
  require(indptr && indices && info, MG_ERR_INPUT, "NULL argument");
  HostPlan hp;
  std::vector<int> lidx;
  host_plan(n, indptr, indices, nranks, rank, hp, local_indices ? &lidx : nullptr);
  info->r0 = hp.r0;
  info->nloc = hp.nloc;
  info->nhalo = (int64_t)hp.halo.size();
  info->nsend = (int64_t)hp.send_rows.size();
  info->local_nnz = indptr[hp.r0 + hp.nloc] - indptr[hp.r0];
  if (halo) std::copy(hp.halo.begin(), hp.halo.end(), halo);
  if (roff) std::copy(hp.roff.begin(), hp.roff.end(), roff);
  if (rcnt) std::copy(hp.rcnt.begin(), hp.rcnt.end(), rcnt);
  if (soff) std::copy(hp.soff.begin(), hp.soff.end(), soff);
  if (scnt) std::copy(hp.scnt.begin(), hp.scnt.end(), scnt);
  if (send_rows) std::copy(hp.send_rows.begin(), hp.send_rows.end(), send_rows);
  if (local_indices) std::copy(lidx.begin(), lidx.end(), local_indices);
  MG_API_END
}

int mg_embed_host(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *weights, int32_t K, const mg_solver_cfg *cfg,
                  int32_t literal_diagonal, int32_t require_convergence, int32_t check_connected,
                  const double *normals, int64_t n_normals, double *P, double *b,
                  mg_solver_out *out, mg_embed_diag *diag) {
  MG_API_BEGIN(ctx)
  require(cfg != nullptr, MG_ERR_INPUT, "cfg is NULL");
  int64_t nnz = indptr[n];
  DBuf<int64_t> dptr(ctx, n + 1), didx(ctx, nnz > 0 ? nnz : 1);
  DBuf<double> dw(ctx, nnz > 0 ? nnz : 1), dz(ctx, n_normals > 0 ? n_normals : 1);
  MG_CUDA(cudaMemcpyAsync(dptr.p, indptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                          ctx->stream));
  MG_CUDA(cudaMemcpyAsync(didx.p, indices, nnz * sizeof(int64_t), cudaMemcpyHostToDevice,
                          ctx->stream));
  MG_CUDA(cudaMemcpyAsync(dw.p, weights, nnz * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  MG_CUDA(cudaMemcpyAsync(dz.p, normals, n_normals * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  // reserved == 1 returns all K+1 pairs (the header's P / eigenvalues sizes)
  const int64_t ncol = (int64_t)K + (cfg->reserved == 1 ? 1 : 0);
  DBuf<double> dP(ctx, n * ncol), db(ctx, n);
  int rc = MG_OK;
  std::string msg;
  try {
    embed_impl(ctx, n, dptr.p, didx.p, dw.p, K, cfg, literal_diagonal, require_convergence,
               check_connected, dz.p, n_normals, dP.p, db.p, out, diag);
  } catch (const Error &e) {
    if (e.code != MG_ERR_NOT_CONVERGED) throw;
    rc = e.code;
    msg = e.what();
  }
  MG_CUDA(cudaMemcpyAsync(P, dP.p, n * ncol * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  MG_CUDA(cudaMemcpyAsync(b, db.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (rc != MG_OK) throw Error(rc, msg);
  MG_API_END
}

}  // extern "C"
