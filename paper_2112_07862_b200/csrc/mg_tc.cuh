// Tensor-core (tcgen05, kind::tf32) Gram pair for the fp32 solve at wide
// blocks (K = 16 / 32: w = 3mp = 60 ... 108 columns), where the CUDA-core
// k_gram2 is FMA-bound (profiles/).
//
//   G_B = S' diag(b) S,  G_A = S' (AS)       S, AS: n x ld row-major fp32
//
// fp32 accuracy from TF32 tensor cores ("3xTF32"): x = hi + lo with
// hi = rna_tf32(x), lo = rna_tf32(x - hi); each product is
// hi*hi + hi*lo + lo*hi (relative error ~2^-21).  The MMA accumulates 64 rows
// in fp32 TMEM, then the epilogue folds the tile into an error-compensated
// fp32 pair per entry (Fast2Sum), and the CTA partial is written in fp64.
//
// Work split: CTA pair (2c, 2c+1) owns a contiguous row range; CTA 2c+h
// computes columns [h*nh, h*nh + nh) of both Grams for ALL w rows
// (M = 128 lanes, N = 64 columns per Gram), so the fp64-accurate accumulators
// (2 x 64 fp32 pairs per thread) fit the register file.  The pair reads the
// same rows concurrently (L2 hits for the second reader).
//
// 8 warps (2 per SM sub-partition: the 2 x 64 accumulator pairs need the
// full 255-register budget).  All warps convert raw fp32 rows into hi/lo
// operand tiles (canonical no-swizzle K-major layout) and drain TMEM; thread 0
// also issues the bulk row copies and the tcgen05.mma stream.  Pipelines: raw
// ring (2 stages, cp.async.bulk + mbarrier), operand ring (2 stages, freed by
// tcgen05.commit), TMEM accumulators (2 buffers x 128 columns).
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

// fast-path update on the tensor cores (fp32 wide blocks): P = S Zp, X = S Zx
// (and A-images), residual W and column partials; returns the CTA count
bool update_tc_supported(int w, int mp);
int update_tc(mg_ctx *ctx, int64_t n, int ld, int w, int m, int mp, float *S, float *AS,
              const float *b, const float *prec, const float *M, const double *theta,
              const int *skip, double *part, float *wc);

}  // namespace mg
