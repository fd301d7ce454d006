// Internal entry points of the operator-construction kernels (mg_graph.cu).
#pragma once
#include "mg_common.cuh"

namespace mg {

int64_t components(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                   int64_t *labels);
void laplacian(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *w,
               int64_t *optr, int64_t *oidx, double *odata);
int64_t two_hop_count(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                      int64_t *tptr);
void two_hop_fill(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                  const int64_t *tptr, int64_t *tidx);
int64_t q_count(mg_ctx *ctx, int64_t n, const int64_t *tptr, int64_t *qptr);
void q_fill(mg_ctx *ctx, int64_t n, const int64_t *tptr, const int64_t *tidx, int literal,
            const int64_t *qptr, int64_t *qidx, double *qdata);
bool check_symmetric(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                     const double *data, double rtol);
double repulsion_weight(mg_ctx *ctx, int64_t n, const int64_t *qptr, const int64_t *qidx,
                        const double *qdata, double eps);
int64_t assemble_count(mg_ctx *ctx, int64_t n, const int64_t *lptr, const int64_t *lidx,
                       const double *ldata, const int64_t *qptr, const int64_t *qidx,
                       const double *qdata, double mu, double eps, int64_t *aptr);
void assemble_fill(mg_ctx *ctx, int64_t n, const int64_t *lptr, const int64_t *lidx,
                   const double *ldata, const int64_t *qptr, const int64_t *qidx,
                   const double *qdata, double mu, double eps, const int64_t *aptr,
                   int64_t *aidx, double *adata);
// returns -1 on success, else the first isolated row (b untouched).  With
// `perm` (row r is original node perm[r]) the reported row and every
// first-index tie-break use original ids.
int64_t degree_balancing(mg_ctx *ctx, int64_t n, const int64_t *aptr, const int64_t *aidx,
                         const double *adata, double *b, double *gdeg,
                         const int64_t *perm = nullptr);
void disc_left_min(mg_ctx *ctx, int64_t n, const int64_t *aptr, const int64_t *aidx,
                   const double *adata, double *min_left, int64_t *row,
                   const int64_t *perm = nullptr);
// Cuthill-McKee locality order (mg_reorder.cu): perm new->old, inv old->new
void cm_order(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, int64_t *perm,
              int64_t *inv);
void permute_graph(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *w,
                   const int64_t *perm, const int64_t *inv, int64_t *nptr, int64_t *nidx,
                   double *nw);
double trace(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *data);
// dense eigenvalues (ascending) of a small CSR matrix, n <= 512 (operators.py:150-152)
void dense_eigvals(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                   const double *data, double *w_host);

// deterministic fp64 reductions over a device array
double sum_f64(mg_ctx *ctx, const double *x, int64_t n);
// numpy's pairwise summation (np.sum of a contiguous float64 array), bit for bit
double np_sum_f64(mg_ctx *ctx, const double *x, int64_t n);
// sqrt(np.sum(data * data)) (sparse.py:76-77)
double frobenius_np(mg_ctx *ctx, const double *data, int64_t nnz);
// mg_queries.cu: sequential row sums; Gershgorin centers / radii / left ends
// (any output may be null); balance_radii (operators.py:189-202)
void row_sums(mg_ctx *ctx, int64_t n, const int64_t *ptr, const double *v, double *out);
void gershgorin(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *v,
                double *center, double *radius, double *left);
void balance_radii(mg_ctx *ctx, int64_t n, const double *radii, double *b, double *gdeg,
                   const int64_t *perm = nullptr);
double max_f64_const(mg_ctx *ctx, const double *x, int64_t n);

}  // namespace mg
