// Device k-means / normalize_rows (clustering.py:50-134, rng.py:9-127).
#pragma once
#include "mg_common.cuh"

namespace mg {
// X: device n x d row-major fp64; labels_out: device int64[n]; returns the
// winning restart's within-cluster sum of squares
double kmeans(mg_ctx *ctx, int64_t n, int d, const double *X, int c, int restarts, uint64_t seed,
              int64_t *labels_out);
void normalize_rows(mg_ctx *ctx, int64_t n, int d, const double *X, double *Y);
}  // namespace mg
