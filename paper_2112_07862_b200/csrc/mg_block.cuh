// Tall-skinny block kernels of the LOBPCG loop (device side of
// eigensolver.py:156-283) and the solver interface used by mg_embed.
#pragma once
#include "mg_common.cuh"

namespace mg {
struct Comm;

template <typename T>
struct VecT;
template <>
struct VecT<float> {
  using V = float4;
  static constexpr int N = 4;
};
template <>
struct VecT<double> {
  using V = double2;
  static constexpr int N = 2;
};

// Solver-side CSR: int64 row pointers, int32 column ids, T values.
template <typename T>
struct DevCSR {
  int64_t n = 0, nnz = 0;
  const int64_t *ptr = nullptr;
  const int *idx = nullptr;
  const T *val = nullptr;
  // fp32 solver: row sums of the fp64 matrix.  A x is then evaluated in
  // difference form  (A x)_i = sum_j A_ij (x_j - x_i) + r_i x_i : the fp32
  // rounding of A_ij becomes a zero-row-sum perturbation whose effect scales
  // with the eigenvalue instead of ||A|| (A and Q are Laplacian-like).
  const T *rowsum = nullptr;
};

// Owning version (conversion from the reference's int64/f64 CSR).
template <typename T>
struct OwnedCSR {
  DBuf<int64_t> ptr;
  DBuf<int> idx;
  DBuf<T> val;
  DBuf<T> rowsum;
  DevCSR<T> view;
};

template <typename T>
void make_solver_csr(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx,
                     const double *val, OwnedCSR<T> &out, int64_t nnz_hint = -1);

// Y[:, 0:w) = A * X[:, 0:w), w a multiple of VecT<T>::N, row-major with lds.
template <typename T>
void spmm(mg_ctx *ctx, const DevCSR<T> &A, const T *X, int ldx, T *Y, int ldy, int w);

struct SolveSpec {
  int k = 1;
  int max_iter = 500;
  double tol = 1e-8;
  bool jacobi = true;
  const double *normals = nullptr;  // device, standard-normal stream
  int64_t n_normals = 0;
  const double *deflate = nullptr;  // device: n_deflate vectors (vector j at deflate + j * deflate_ld) or null
  int n_deflate = 1;
  int64_t deflate_ld = 0;
  const int64_t *perm = nullptr;    // optional: solver row r is original row perm[r]
  // distributed mode (mg_dist.cuh): communicator and this rank's DistPart<T>;
  // rows are the global rows [row_base, row_base + n_local)
  struct Comm *comm = nullptr;
  const void *dist = nullptr;
  int64_t row_base = 0;
  int64_t n_global = 0;
};

struct SolveResult {
  std::vector<double> eigenvalues, residual_norms, history;
  std::vector<int> converged;
  int iterations = 0;
  int64_t normals_used = 0;
  int64_t fast_steps = 0, fast_fallbacks = 0;
};

// lobpcg_smallest on (A, diag(b)); eigvecs: device n x k double row-major in
// ORIGINAL row order (if spec.perm is set, row perm[r] <- solver row r).
template <typename T>
SolveResult lobpcg(mg_ctx *ctx, const DevCSR<T> &A, double anorm, const double *b_dev,
                   const double *diagA_dev, const SolveSpec &spec, double *eigvecs);

}  // namespace mg
