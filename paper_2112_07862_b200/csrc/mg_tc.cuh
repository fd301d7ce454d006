// Tensor-core (tcgen05, kind::tf32) Gram pair for the fp32 solve at wide
// blocks (K = 16 / 32: w = 3mp = 60 ... 108 columns), where the CUDA-core
// k_gram2 is FMA-bound:
//
//   G_B = S' diag(b) S,  G_A = S' (AS)       S, AS: n x ld row-major fp32
//
// The kernel (mg_tc2.cu) is TMA-fed with a 2-piece TF32 split; design notes
// at the top of that file.
#pragma once
#include "mg_common.cuh"

namespace mg {

// host side (mg_tc.cu)
bool gram_tc_supported(int w);
// G_B / G_A (w x w, row-major fp64) of fp32 S, AS (n x ld) with weights b
void gram_pair_tc(mg_ctx *ctx, int64_t n, int ld, int w, const float *S, const float *AS,
                  const float *b, double *GB, double *GA, DBuf<double> &part);

// v2 (mg_tc2.cu): TMA-fed, SW128 MN-major operands, one CTA per SM
bool gram_tc2_supported(int w, int ld);
void gram_pair_tc2(mg_ctx *ctx, int64_t n, int ld, int w, const float *S, const float *AS,
                   const float *b, double *GB, double *GA, DBuf<double> &part);

// narrow mode of the same kernel: only the W-column blocks of both Grams
bool gram_w_tc2_supported(int w, int mp, int ld);
void gram_w_tc2(mg_ctx *ctx, int64_t n, int ld, int w, int mp, const float *S, const float *AS,
                const float *b, double *GB, double *GA, DBuf<double> &part);

// tcgen05 update (mg_tc3.cu): P = S Zp, X += S (Zp + [Yx - I; 0; 0]) and the
// A-images, fused residual / W / column norms; returns the grid (rows of part)
bool update_tc3_supported(int w, int mp, int ld);
int update_tc3(mg_ctx *ctx, int64_t n, int ld, int w, int m, int mp, float *S, float *AS,
               const float *b, const float *prec, const float *Mg, const double *theta,
               const int *skip, double *part, float *wc, const int *perm, int wc0, int wcs);
void update_f32_hook(mg_ctx *ctx, int variant, int64_t n, int ld, int m, int mp, float *S,
                     float *AS, const float *b, const float *prec, const float *Mg,
                     const double *theta, float *wc, double *colsums);

}  // namespace mg
