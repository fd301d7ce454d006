/*
 * manigraph_b200.h -- C ABI of the B200-native (A, B) formation + LOBPCG path.
 *
 * Drop-in boundary for the reference package `manigraph` (pure Python; its
 * public API is re-exported at /root/reference/pkg/src/manigraph/__init__.py
 * :23-66).  Every entry point below replaces one reference function; the
 * citation names the function and file:line it replaces.  The reference has
 * no FFI of its own, so the binding a maintainer would add is a ctypes shim
 * (INTEGRATION.md shows it; paper_2112_07862_b200/_native.py is that shim).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Unless a parameter says "host", array
 *    pointers are CUDA DEVICE pointers on the context's device.
 *  - CSR matrices: indptr int64[n+1], indices int64[nnz] (sorted, unique per
 *    row), data double[nnz]  (the reference dtypes, sparse.py:25-27).
 *  - Block vectors are row-major n x k double arrays (numpy C order, the
 *    layout of the reference's `eigenvectors` arrays).
 *  - Work is stream-ordered on the context's stream; every call returns after
 *    its results are complete (blocking from the caller's view, like the
 *    reference's synchronous Python calls).
 *  - Outputs of data-dependent size use a two-phase protocol: a *_count call
 *    fills indptr and returns nnz on the host, the caller allocates, then the
 *    *_fill call writes indices/data.
 *  - Return value: an mg_status code.  mg_last_error() returns a thread-local
 *    message for the last failing call on this thread.  Codes map to the
 *    reference exceptions (errors.py:6-45): MG_ERR_INPUT -> InputError,
 *    MG_ERR_DISCONNECTED -> DisconnectedGraphError, MG_ERR_NOT_CONVERGED ->
 *    ConvergenceError (outputs are still filled, best effort).
 */
#ifndef MANIGRAPH_B200_H
#define MANIGRAPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mg_status {
  MG_OK = 0,
  MG_ERR_INPUT = 1,
  MG_ERR_DISCONNECTED = 2,
  MG_ERR_NOT_CONVERGED = 3,
  MG_ERR_CUDA = 4,
  MG_ERR_NCCL = 5,
  MG_ERR_NOMEM = 6,
  MG_ERR_INTERNAL = 7,
  MG_ERR_PARSE = 8 /* -> ParseError (errors.py:14-20); see mg_load_edge_list_count */
} mg_status;

typedef struct mg_ctx mg_ctx;

/* ---- library / context ------------------------------------------------- */
int mg_version(void);                                  /* ABI version */
const char *mg_last_error(void);                       /* thread-local */
int mg_device_count(int *count /* host */);
/* stream: a cudaStream_t or NULL for a library-owned stream */
int mg_ctx_create(int device, void *stream, mg_ctx **out);
int mg_ctx_destroy(mg_ctx *ctx);
int mg_ctx_set_stream(mg_ctx *ctx, void *stream);
/* Number of native kernel launches issued through this context so far. */
int mg_ctx_launch_count(mg_ctx *ctx, int64_t *count /* host */);
/* The cudaStream_t the context issues work on (for caller-side CUDA events). */
int mg_ctx_get_stream(mg_ctx *ctx, void **stream /* host */);

/* Hot-kernel timing: when enabled, CUDA events bracket every SpMM / Gram /
 * update / residual / control launch.  mg_ctx_stats aggregates (and clears)
 * them per class: counts[c], milliseconds[c], algorithmic bytes[c] for
 * c = 0 spmm, 1 gram, 2 update, 3 resid, 4 ctrl, 5 setup. */
int mg_ctx_set_profiling(mg_ctx *ctx, int enable);
int mg_ctx_stats(mg_ctx *ctx, int64_t *counts /* host 6 */, double *milliseconds /* host 6 */,
                 double *bytes /* host 6 */);

/* ---- graph-level pieces -------------------------------------------------- */
/* Graph.connected_components (graph.py:107-123): count + labels numbered by
 * each component's smallest node id (the reference's DFS scan order). */
int mg_components(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  int64_t *labels /* device n, may be NULL */, int64_t *count /* host */);

/* laplacian (graph.py:321-346) incl. degrees (graph.py:93-96).  Output nnz is
 * always nnz(graph) + n; out_indptr n+1. */
int mg_laplacian(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                 const double *weights, int64_t *out_indptr, int64_t *out_indices,
                 double *out_data);

/* two_hop_sets (operators.py:88-108): pattern(adj@adj) - diag - pattern(adj). */
int mg_two_hop_count(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                     int64_t *t_indptr /* n+1 */, int64_t *t_nnz /* host */);
int mg_two_hop_fill(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const int64_t *t_indptr, int64_t *t_indices);

/* two_hop_laplacian (operators.py:111-135). */
int mg_two_hop_laplacian_count(mg_ctx *ctx, int64_t n, const int64_t *t_indptr,
                               int64_t *q_indptr /* n+1 */, int64_t *q_nnz /* host */);
int mg_two_hop_laplacian_fill(mg_ctx *ctx, int64_t n, const int64_t *t_indptr,
                              const int64_t *t_indices, int literal_diagonal,
                              const int64_t *q_indptr, int64_t *q_indices, double *q_data);

/* SparseSymMatrix.check_symmetric (sparse.py:100-105): *is_symmetric = 0/1. */
int mg_check_symmetric(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                       const double *data, double rtol, int *is_symmetric /* host */);

/* repulsion_weight (operators.py:159-176); returns MG_ERR_INPUT for eps < 0. */
int mg_repulsion_weight(mg_ctx *ctx, int64_t n, const int64_t *q_indptr,
                        const int64_t *q_indices, const double *q_data, double epsilon,
                        double *mu /* host */);

/* assemble_operator (operators.py:179-186): (L - mu*Q) + eps*I with exact-zero
 * dropping and the reference's separate roundings. */
int mg_assemble_count(mg_ctx *ctx, int64_t n, const int64_t *l_indptr, const int64_t *l_indices,
                      const double *l_data, const int64_t *q_indptr, const int64_t *q_indices,
                      const double *q_data, double mu, double epsilon,
                      int64_t *a_indptr /* n+1 */, int64_t *a_nnz /* host */);
int mg_assemble_fill(mg_ctx *ctx, int64_t n, const int64_t *l_indptr, const int64_t *l_indices,
                     const double *l_data, const int64_t *q_indptr, const int64_t *q_indices,
                     const double *q_data, double mu, double epsilon, const int64_t *a_indptr,
                     int64_t *a_indices, double *a_data);

/* degree_balancing (operators.py:205-219) + balance_radii (189-202) +
 * SparseSymMatrix.gershgorin (sparse.py:84-94).  On MG_ERR_DISCONNECTED
 * *isolated_node holds the first row with radius <= 0. */
int mg_degree_balancing(mg_ctx *ctx, int64_t n, const int64_t *a_indptr,
                        const int64_t *a_indices, const double *a_data, double *b /* device n */,
                        double *generalized_degree /* host */, int64_t *isolated_node /* host */);

/* SparseSymMatrix.row_sums (sparse.py:79-82) and Graph.degrees
 * (graph.py:93-96): per-row sums in stored order; out device n. */
int mg_row_sums(mg_ctx *ctx, int64_t n, const int64_t *indptr, const double *data, double *out);

/* SparseSymMatrix.gershgorin / disc_left_ends (sparse.py:84-98): centers =
 * stored diagonal, radii = off-diagonal |a_ij| summed in stored order, left
 * ends = centers - radii; each output device n, or NULL to skip. */
int mg_gershgorin(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *data, double *centers, double *radii, double *left_ends);

/* SparseSymMatrix.frobenius_norm (sparse.py:76-77): sqrt of numpy's pairwise
 * sum of the squared values, bit for bit; out host. */
int mg_frobenius_norm(mg_ctx *ctx, int64_t nnz, const double *data, double *out);

/* balance_radii (operators.py:189-202): b device n, generalized_degree host. */
int mg_balance_radii(mg_ctx *ctx, int64_t n, const double *radii, double *b,
                     double *generalized_degree);

/* OperatorPair.diagnostics (operators.py:76-85): min disc left end + row. */
int mg_disc_left_min(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
                     const double *a_data, double *min_left /* host */,
                     int64_t *binding_row /* host */);

/* ---- eigensolver ----------------------------------------------------------- */
typedef struct mg_solver_cfg {
  int32_t k;               /* block size (SolverConfig.k, eigensolver.py:32-48) */
  int32_t max_iter;
  double tol;
  int32_t preconditioner;  /* 0 none, 1 jacobi */
  int32_t precision;       /* 0 fp64, 1 fp32 vectors with fp64 Gram/Rayleigh-Ritz */
  int32_t reorder;         /* 1: locality reordering of rows inside the solve */
  int32_t reserved;        /* mg_embed only: 1 = return all K+1 pairs in P/eigenvalues */
} mg_solver_cfg;

typedef struct mg_solver_out {
  /* mg_lobpcg: k entries each.  mg_embed / mg_embed_host: eigenvalues K
   * (K+1 with cfg->reserved == 1); residual_norms and converged always K+1
   * (the solver's view, including the dropped pair). */
  double *eigenvalues;      /* host */
  double *residual_norms;   /* host */
  int32_t *converged;       /* host */
  double *history;          /* host, capacity history_cap (ritz_sum_history) */
  int32_t history_cap;
  int32_t iterations;       /* out */
  int32_t history_len;      /* out */
  int32_t normals_used;     /* out: entries consumed from the normal stream */
} mg_solver_out;

/* lobpcg_smallest (eigensolver.py:156-283).  `normals` is the seeded standard
 * normal stream (numpy PCG64(seed).standard_normal order): the initial block
 * is normals[0 : n*k] read as n x k row-major, refills continue the stream
 * (eigensolver.py:177-178, 189).  `deflate` (device n, or NULL) is one vector
 * projected out in the B inner product (eigensolver.py:179-184, 239-241).
 * eigenvectors: device n x k row-major.  Returns MG_OK even when not all
 * pairs converged (check out->converged), like the reference. */
int mg_lobpcg(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
              const double *a_data, const double *b, const mg_solver_cfg *cfg,
              const double *normals, int64_t n_normals, const double *deflate,
              double *eigenvectors, mg_solver_out *out);

/* lobpcg_smallest with several deflation vectors (eigensolver.py:179-184,
 * 189-192, 239-241: `for col in defl.T: block = _b_project_out(col, block)`).
 * `deflate` is device n x n_deflate COLUMN-major (vector j at deflate + j*n);
 * the vectors are projected out one after another in that order, exactly as
 * the reference does (no joint orthogonalisation).  mg_lobpcg is the
 * n_deflate <= 1 case. */
int mg_lobpcg_deflate(mg_ctx *ctx, int64_t n, const int64_t *a_indptr, const int64_t *a_indices,
                      const double *a_data, const double *b, const mg_solver_cfg *cfg,
                      const double *normals, int64_t n_normals, const double *deflate,
                      int32_t n_deflate, double *eigenvectors, mg_solver_out *out);

/* smallest_above_null (eigensolver.py:431-460) as used by identity_shift
 * (operators.py:138-156): smallest eigenvalue of Q above tau = 1e-8 tr(Q)/n,
 * dense for n <= 512, else deflated LOBPCG (k = 8 doubling to 64, tol 1e-6,
 * 60 iterations).  Includes check_symmetric (MG_ERR_INPUT if asymmetric). */
int mg_identity_shift(mg_ctx *ctx, int64_t n, const int64_t *q_indptr,
                      const int64_t *q_indices, const double *q_data,
                      const double *normals, int64_t n_normals, int32_t precision,
                      double *epsilon /* host */);

/* smallest_above_null (eigensolver.py:431-460) with explicit tau/tol/max_iter
 * (fiedler_value, eigensolver.py:463-468, uses tol 1e-8 / 500).  No symmetry check. */
int mg_smallest_above_null(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                           const double *data, double tau, double tol, int32_t max_iter,
                           const double *normals, int64_t n_normals, int32_t precision,
                           double *value /* host */);

/* SparseSymMatrix.matmat (sparse.py:67-68): Y = A X, X/Y device n x k row-major. */
int mg_spmm(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
            const double *data, const double *X, int32_t k, double *Y);

/* ---- end-to-end ------------------------------------------------------------ */
typedef struct mg_embed_diag {
  double mu, epsilon, min_disc_left_end, dropped_eigenvalue, generalized_degree;
  int64_t binding_row, q_nnz, a_nnz, t_nnz, n_components;
  int32_t iterations, eps_iterations;
  double seconds_setup, seconds_eps, seconds_solve;
  int64_t fast_steps, fast_fallbacks;   /* single-Gram-pass iterations / fallbacks */
} mg_embed_diag;

/* embed (embedding.py:77-103): components check, build_operator_pair,
 * K+1-pair LOBPCG, drop the first pair.  P: device n x K row-major (n x (K+1)
 * with cfg->reserved == 1); eigenvalues host K (K+1); b device n.  `normals`
 * as in mg_lobpcg: the eps solve may double its block from 8 to 64 and
 * refills continue the stream, so pass at least n * max(K+1, 64) entries
 * plus a refill margin; a short stream fails with MG_ERR_INPUT ("normal
 * stream exhausted") and the caller retries with a longer one (core.embed
 * does).  check_connected = 0 bypasses the component test
 * (SURVEY F6, config 4).  Returns MG_ERR_NOT_CONVERGED (outputs filled) when
 * require_convergence and some pair is unconverged. */
int mg_embed(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
             const double *weights, int32_t K, const mg_solver_cfg *cfg,
             int32_t literal_diagonal, int32_t require_convergence, int32_t check_connected,
             const double *normals, int64_t n_normals, double *P, double *b,
             mg_solver_out *out, mg_embed_diag *diag);

/* Same as mg_embed with HOST input/output arrays (library allocates device
 * memory; host<->device copies happen inside). */
int mg_embed_host(mg_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *weights, int32_t K, const mg_solver_cfg *cfg,
                  int32_t literal_diagonal, int32_t require_convergence,
                  int32_t check_connected, const double *normals, int64_t n_normals,
                  double *P, double *b, mg_solver_out *out, mg_embed_diag *diag);

/* Gram pair of the fp32 solve on the tensor cores (tcgen05, 3xTF32):
 * GB = S' diag(b) S, GA = S' AS over the first w columns of row-major n x ld
 * fp32 blocks (48 < w <= 128, ld % 4 == 0); outputs w x w row-major fp64.
 * Replaces, in one pass over the block, the B-inner products of the
 * reference's _b_mgs_pair (eigensolver.py:127, 143, 145: prefix.T @ (b*rest),
 * U.T @ (b*v), v @ (b*v)) and the Rayleigh-Ritz Gram S.T @ AS
 * (eigensolver.py:251), at the K = 16..32 block widths. */
int mg_gram_pair_f32(mg_ctx *ctx, int64_t n, int32_t ld, int32_t w, const float *S,
                     const float *AS, const float *b, double *GB, double *GA);

/* One LOBPCG basis update of the fp32 solve, in place on row-major n x ld
 * fp32 blocks S = [X | P | W] and AS = [AX | AP | AW] (column blocks of width
 * mp, m <= mp real columns), eigensolver.py:255-266:
 *   P = S Zp, X = X Yx + P, AP = AS Zp, AX = AX Yx + AP,
 *   R = AX - b X Theta (eigensolver.py:225), W = prec R (eigensolver.py:239),
 * M = [Zp (3mp x mp) ; Yx (mp x mp)] row-major fp32, theta fp64 (m), prec may
 * be NULL.  W is also written to the compact n x mp block wc (the SpMM input).
 * colsums (2 mp, fp64): sum R^2 per column, then sum X^2 per column.
 * variant 0: fp32 FMA kernel; variant 1: tcgen05 (3 mp <= 128), which forms
 * only the corrections X (Yx - I) + P on the tensor core and adds them to the
 * old X / AX in fp32. */
int mg_update_f32(mg_ctx *ctx, int32_t variant, int64_t n, int32_t ld, int32_t m, int32_t mp,
                  float *S, float *AS, const float *b, const float *prec, const float *M,
                  const double *theta, float *wc, double *colsums);

/* Host <-> device copies for large pageable host buffers (results, inputs):
 * pipelined through the context's pinned stages; blocking. */
int mg_copy_d2h(mg_ctx *ctx, void *host, const void *dev, int64_t bytes);
int mg_copy_h2d(mg_ctx *ctx, void *dev, const void *host, int64_t bytes);

/* numpy's Generator(PCG64).standard_normal stream, bit for bit, on the device:
 * the reference's initial block (eigensolver.py:177-178, 189) is the first
 * n*m values of default_rng(seed).standard_normal.  (state, inc) are the 128-bit
 * halves of default_rng(seed).bit_generator.state['state']; out: device double[count]. */
int mg_normal_stream(mg_ctx *ctx, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, int64_t count, double *out);

/* ---------------------------------------- text I/O -------
 * Host arrays, host files; the same bytes as the reference writers and the
 * same values / errors as its readers.  threads <= 0: all host cores. */
/* save_embedding_csv (embedding.py:131-140): "node,c1,...,cK" + rows "i,v,..."
 * with format(v, '.17g'); P row-major n x k */
int mg_save_embedding_csv(const char *path, int64_t n, int32_t k, const double *P,
                          int32_t threads);
/* load_embedding_csv (embedding.py:143-166): _dims returns (n, k); the fill
 * call writes P (row-major n x k, rows in node-id order) */
int mg_load_embedding_csv_dims(const char *path, int64_t *n, int32_t *k);
int mg_load_embedding_csv(const char *path, int64_t n, int32_t k, double *P, int32_t threads);
/* save_edge_list (graph.py:188-194): "i\tj\tw" for i < j, 17-digit weights */
int mg_save_edge_list(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                      const double *weights, int32_t threads);
/* load_edge_list (graph.py:147-185) -> Graph.from_edges CSR.  _count parses
 * and keeps the result for the calling thread (n, nnz; on MG_ERR_PARSE the
 * 1-based line in *err_line); _fill copies it out (indptr n+1, indices and
 * weights nnz) and releases it. */
int mg_load_edge_list_count(const char *path, int32_t threads, int64_t *n, int64_t *nnz,
                            int64_t *err_line);
int mg_load_edge_list_fill(int64_t *indptr, int64_t *indices, double *weights);

/* ---------------------------------------- binary I/O ------
 * The objects of the text formats above (embedding.py:131-166,
 * graph.py:147-194) as raw little-endian arrays behind a 64-byte header
 * (layout in csrc/mg_binio.cu), written / read by `threads` threads with
 * pwrite / pread (0: hardware concurrency, at most 16).  Host pointers;
 * eigenvalues / b may be NULL.  Loads check the header (MG_ERR_PARSE) and,
 * for graphs, the canonical CSR of Graph.from_edges (MG_ERR_INPUT). */
int mg_save_embedding_bin(const char *path, int64_t n, int32_t k, const double *P,
                          const double *eigenvalues, const double *b, const char *method,
                          int32_t threads);
int mg_load_embedding_bin_dims(const char *path, int64_t *n, int32_t *k, int32_t *has_b,
                               char *method16);
int mg_load_embedding_bin(const char *path, double *P, double *eigenvalues, double *b,
                          int32_t threads);
int mg_save_graph_bin(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                      const double *weights, int32_t threads);
int mg_load_graph_bin_dims(const char *path, int64_t *n, int64_t *nnz);
int mg_load_graph_bin(const char *path, int64_t *indptr, int64_t *indices, double *weights,
                      int32_t threads);

/* --------------------------------------- kNN graph -------
 * knn_graph (graph.py:281-315): symmetrized k-nearest-neighbour graph of the
 * rows of X (device n x d row-major fp64), ties at the k-th distance to the
 * lower index, Gaussian weights exp(-d^2 / sigma^2) with sigma^2 the mean
 * squared distance over the retained edges (weighted != 0), else 1; output
 * in the canonical CSR of Graph.from_edges (graph.py:31-79).  Two-phase:
 * _count fills indptr (device int64[n+1]) and *nnz (host); _fill writes
 * indices (device int64[nnz]) and weights (device double[nnz]).
 * k <= 64, d <= 5120; O(n^2 d) like the reference. */
int mg_knn_graph_count(mg_ctx *ctx, int64_t n, int32_t d, const double *X, int32_t k,
                       int32_t weighted, int64_t *indptr, int64_t *nnz);
int mg_knn_graph_fill(mg_ctx *ctx, int64_t n, int32_t d, const double *X, int32_t k,
                      int32_t weighted, int64_t *indices, double *weights);

/* ------------------------------------------ clustering ---
 * The C4 readout after the embedding: device k-means with the reference's
 * portable seeding streams.  points: device n x d row-major fp64. */
/* kmeans (clustering.py:99-134; k-means++ :57-67, Lloyd :70-96, streams
 * rng.py:9-127): best of `restarts` restarts from xoshiro256** streams
 * stream_seed(seed, r); labels: device int64[n]; wcss: host, may be NULL.
 * d <= 32, c <= 64, c * d <= 512. */
int mg_kmeans(mg_ctx *ctx, int64_t n, int32_t d, const double *points, int32_t c,
              int32_t restarts, uint64_t seed, int64_t *labels, double *wcss);
/* normalize_rows (clustering.py:50-56): unit Euclidean rows, zero rows kept */
int mg_normalize_rows(mg_ctx *ctx, int64_t n, int32_t d, const double *points, double *out);

/* ---------------------------------------------------- multi-GPU (8(e)) ---
 * 1-D row partition of the solve over ranks (one process per GPU).  The
 * setup (Q, eps, mu, A, b) is replicated; each LOBPCG SpMM exchanges halo
 * rows (NCCL grouped send/recv) and every Gram / norm reduction is an NCCL
 * allreduce of a small fp64 block.  The reference has no distributed mode
 * (single-process numpy/scipy, eigensolver.py:165-283); results agree with
 * mg_embed to the solver tolerance (reduction order differs). */
typedef struct mg_comm mg_comm;
int mg_nccl_unique_id(uint8_t *uid /* host 128 bytes */);
int mg_comm_create_nccl(mg_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *uid,
                        mg_comm **out);
/* R virtual ranks as threads of one process (tests; collectives through the host) */
int mg_local_group_create(int32_t nranks, void **group);
int mg_local_group_destroy(void *group);
int mg_comm_create_local(void *group, int32_t rank, mg_comm **out);
int mg_comm_destroy(mg_comm *comm);
/* mg_embed over the ranks of `comm`; every rank passes the full graph and
 * receives the full P / b / diagnostics */
int mg_embed_dist(mg_ctx *ctx, mg_comm *comm, int64_t n, const int64_t *indptr,
                  const int64_t *indices, const double *weights, int32_t K,
                  const mg_solver_cfg *cfg, int32_t literal_diagonal, int32_t require_convergence,
                  int32_t check_connected, const double *normals, int64_t n_normals, double *P,
                  double *b, mg_solver_out *out, mg_embed_diag *diag);
/* halo plan of `rank` for a HOST CSR (no GPU needed): row range [r0, r0+nloc),
 * sorted halo rows, per-peer receive/send offsets+counts (nranks each), local
 * rows to send, and the local CSR's remapped column ids ([local | halo]).
 * Output arrays may be NULL (query sizes via info first). */
typedef struct mg_dist_plan_info {
  int64_t r0, nloc, nhalo, nsend, local_nnz;
} mg_dist_plan_info;
int mg_dist_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, int32_t nranks,
                      int32_t rank, mg_dist_plan_info *info, int64_t *halo, int64_t *roff,
                      int64_t *rcnt, int64_t *soff, int64_t *scnt, int32_t *send_rows,
                      int32_t *local_indices);

#ifdef __cplusplus
}
#endif
#endif /* MANIGRAPH_B200_H */
