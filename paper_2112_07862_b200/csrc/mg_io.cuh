// Text I/O: embedding CSV and edge lists, host C++.
#pragma once
#include <vector>

#include "mg_common.cuh"

namespace mg {
struct EdgeListResult {
  int64_t n = 0, err_line = 0;
  std::vector<int64_t> indptr, indices;
  std::vector<double> weights;
};
void save_embedding_csv(const char *path, int64_t n, int k, const double *P, int threads);
// P == nullptr: dimensions only
void load_embedding_csv(const char *path, int64_t *n, int *k, double *P, int threads);
void save_edge_list(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *w, int threads);
void load_edge_list(const char *path, int threads, EdgeListResult &res);
}  // namespace mg
