// Device kNN graph (graph.py:281-315), SURVEY 8(f).2.
#pragma once
#include "mg_common.cuh"

namespace mg {
struct KnnResult {
  int64_t nnz = 0;
  double sigma2 = 0.0;
  DBuf<int64_t> indptr, indices;
  DBuf<double> weights;
};
// X: device n x d row-major fp64
KnnResult knn_graph(mg_ctx *ctx, int64_t n, int d, const double *X, int k, bool weighted);
}  // namespace mg
