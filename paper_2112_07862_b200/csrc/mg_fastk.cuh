// Fast-path LOBPCG kernels (prefix iterations):
//   k_gram2         one read of S = [X P W] and AS -> G_B = S'BS and G_A = S'AS
//   k_ctrl_fast     two-pass projection + Cholesky (drop rule) + Rayleigh-Ritz
//                   entirely on the small Gram matrices (one thread block)
//   k_update_resid  P = S Zp, X = X Yx + P (and A-images), then the next
//                   residual block W = dinv (AX - B X Theta) and its norms
// Row tiles of S/AS are staged with 1-D bulk async copies (cp.async.bulk +
// mbarrier complete_tx) into a shared-memory ring.
#pragma once
#include "mg_block.cuh"
#include "mg_small.cuh"
#include "mg_eig.cuh"

namespace mg {

static constexpr int kFTK = 32;      // rows per tile
static constexpr int kMaxFast = 256;
static constexpr int kFThreads = 256;

// ------------------------------------------------------- bulk copy helpers ---
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// issue the copies of row tile `tile` (rows [tile*tk, ...)) into ring stage st
template <typename T>
__device__ __forceinline__ void issue_tile(const T *S, const T *AS, const T *b, int64_t n, int ld,
                                           int tk, int64_t tile, T *sS, T *sA, T *sb,
                                           uint64_t *bar) {
  int64_t r0 = tile * tk;
  int nr = (int)min((int64_t)tk, n - r0);
  uint32_t bytes_m = (uint32_t)(nr * ld * sizeof(T));
  uint32_t bytes_b = (uint32_t)(((nr * sizeof(T)) + 15) / 16 * 16);
  uint32_t total = bytes_m * (AS ? 2 : 1) + (b ? bytes_b : 0);
  mbar_expect_tx(bar, total);
  bulk_g2s(sS, S + r0 * ld, bytes_m, bar);
  if (AS) bulk_g2s(sA, AS + r0 * ld, bytes_m, bar);
  if (b) bulk_g2s(sb, b + r0, bytes_b, bar);
}

// ------------------------------------------------------------- k_gram2 ---
// Thread layout: nbr Gram blocks (8x8) in this round; groups of nbr threads
// split the rows of each tile (row r -> group r % G).  fp32 data: products
// accumulate in fp32 over a few tiles, then flush into fp64 (shared memory);
// fp64 data accumulates in fp64 registers.
struct Gram2Args {
  int64_t n;
  int tk;                 // rows per tile
  int ld, w, nb;          // w columns [0, w), nb = ceil(w/8) blocks per side
  int blk_lo, nbr;        // Gram blocks [blk_lo, blk_lo + nbr) of the enumeration
  int nsym;               // blocks per Gram: nb*(nb+1)/2
  double *part;           // [grid][2][w*w] (only computed block entries written)
};

__device__ __forceinline__ void gram2_decode(int blk, int nb, int nsym, int &g, int &bi, int &bj) {
  g = blk >= nsym ? 1 : 0;
  int t = blk - g * nsym;
  int r = 0;
  while (t >= nb - r) {
    t -= nb - r;
    ++r;
  }
  bi = r;
  bj = r + t;
}

template <typename T, int NS>
__global__ void __launch_bounds__(kFThreads, 1)
    k_gram2(const T *__restrict__ S, const T *__restrict__ AS, const T *__restrict__ b,
            Gram2Args a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr bool F32 = sizeof(T) == 4;
  const int ld = a.ld, TK = a.tk;
  const size_t tile_elems = (size_t)TK * ld + 16;
  T *ring = reinterpret_cast<T *>(smraw);
  // stage s: S tile, AS tile, b tile
  auto stS = [&](int s) { return ring + (size_t)s * (2 * tile_elems + TK + 16); };
  auto stA = [&](int s) { return stS(s) + tile_elems; };
  auto stB = [&](int s) { return stS(s) + 2 * tile_elems; };
  unsigned char *after = smraw + (size_t)NS * (2 * tile_elems + TK + 16) * sizeof(T);
  after = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(after) + 15) & ~uintptr_t(15));
  uint64_t *bars = reinterpret_cast<uint64_t *>(after);
  double *acc64 = reinterpret_cast<double *>(after + 64);  // [64][kFThreads]

  const int tid = threadIdx.x;
  const int G = max(1, kFThreads / a.nbr);
  const int grp = tid / a.nbr, blk = tid - grp * a.nbr;
  const bool active = grp < G;
  int g = 0, bi = 0, bj = 0;
  if (active) gram2_decode(a.blk_lo + blk, a.nb, a.nsym, g, bi, bj);

  const int64_t ntiles = (a.n + TK - 1) / TK;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_proxy_async();
  }
  if (F32)
    for (int e = tid; e < 64 * kFThreads; e += kFThreads) acc64[e] = 0.0;
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < NS && t_begin + s < t_end; ++s)
      issue_tile(S, AS, b, a.n, ld, TK, t_begin + s, stS(s), stA(s), stB(s), &bars[s]);

  float accf[64];
  double accd[F32 ? 1 : 64];
#pragma unroll
  for (int e = 0; e < 64; ++e) accf[e] = 0.f;
  if (!F32) {
#pragma unroll
    for (int e = 0; e < (F32 ? 1 : 64); ++e) accd[e] = 0.0;
  }
  int since_flush = 0;
  for (int64_t t = t_begin; t < t_end; ++t) {
    const int s = (int)((t - t_begin) % NS);
    const uint32_t phase = (uint32_t)(((t - t_begin) / NS) & 1);
    mbar_wait(&bars[s], phase);
    const int nr = (int)min((int64_t)TK, a.n - t * TK);
    if (active) {
      const T *U = stS(s) + bi * 8;
      const T *Vb = (g == 0 ? stS(s) : stA(s)) + bj * 8;
      const T *bb = stB(s);
      for (int r = grp; r < nr; r += G) {
        T u[8], v[8];
        if constexpr (F32) {
          const float4 u0 = reinterpret_cast<const float4 *>(U + r * ld)[0];
          const float4 u1 = reinterpret_cast<const float4 *>(U + r * ld)[1];
          const float4 v0 = reinterpret_cast<const float4 *>(Vb + r * ld)[0];
          const float4 v1 = reinterpret_cast<const float4 *>(Vb + r * ld)[1];
          u[0] = u0.x; u[1] = u0.y; u[2] = u0.z; u[3] = u0.w;
          u[4] = u1.x; u[5] = u1.y; u[6] = u1.z; u[7] = u1.w;
          v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w;
          v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
        } else {
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const double2 uu = *reinterpret_cast<const double2 *>(U + r * ld + q);
            const double2 vv = *reinterpret_cast<const double2 *>(Vb + r * ld + q);
            u[q] = uu.x; u[q + 1] = uu.y;
            v[q] = vv.x; v[q + 1] = vv.y;
          }
        }
        if (g == 0) {
          const T wr = bb[r];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = wr * v[q];
        }
        if (F32) {
#pragma unroll
          for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) accf[x * 8 + y] = fmaf((float)u[x], (float)v[y], accf[x * 8 + y]);
        } else {
#pragma unroll
          for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y)
              accd[(x * 8 + y) % (F32 ? 1 : 64)] =
                  fma((double)u[x], (double)v[y], accd[(x * 8 + y) % (F32 ? 1 : 64)]);
        }
      }
    }
    __syncthreads();  // everyone is done with stage s
    if (tid == 0 && t + NS < t_end) {
      fence_proxy_async();
      issue_tile(S, AS, b, a.n, ld, TK, t + NS, stS(s), stA(s), stB(s), &bars[s]);
    }
    since_flush += (nr + G - 1) / G;  // rows this thread accumulated in fp32
    if (F32 && since_flush >= 32) {
      since_flush = 0;
      if (active) {
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          acc64[e * kFThreads + tid] += (double)accf[e];
          accf[e] = 0.f;
        }
      }
    }
  }
  if (F32) {
    if (active) {
#pragma unroll
      for (int e = 0; e < 64; ++e) acc64[e * kFThreads + tid] += (double)accf[e];
    }
  } else {
    if (active) {
#pragma unroll
      for (int e = 0; e < (F32 ? 1 : 64); ++e) acc64[e * kFThreads + tid] = accd[e];
    }
  }
  __syncthreads();
  // reduce the row groups (fixed order) and write this CTA's partial Grams
  const int w = a.w;
  double *dst = a.part + (size_t)blockIdx.x * 2 * w * w;
  for (int item = tid; item < a.nbr * 64; item += kFThreads) {
    const int bk = item / 64, e = item - bk * 64;
    double sum = 0.0;
    for (int q = 0; q < G; ++q) sum += acc64[e * kFThreads + q * a.nbr + bk];
    int gg, ii, jj;
    gram2_decode(a.blk_lo + bk, a.nb, a.nsym, gg, ii, jj);
    const int i = ii * 8 + (e >> 3), j = jj * 8 + (e & 7);
    if (i < w && j < w) dst[(size_t)gg * w * w + i * w + j] = sum;
  }
}

// sum CTA partials (fixed order) and mirror the symmetric lower blocks
static __global__ void k_reduce_gram2(const double *__restrict__ part, int nb_cta, int w,
                               double *__restrict__ GB, double *__restrict__ GA) {
  const int tot = 2 * w * w;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int g = e / (w * w);
    const int r = e - g * w * w;
    int i = r / w, j = r - i * w;
    if ((i >> 3) > (j >> 3)) {
      int t = i;
      i = j;
      j = t;
    }
    const size_t src = (size_t)g * w * w + i * w + j;
    double s = 0.0;
    for (int q = 0; q < nb_cta; ++q) s += part[(size_t)q * tot + src];
    (g ? GA : GB)[r] = s;
  }
}

// -------------------------------------------------------- k_update_resid ---
// P_new = S[:, 0:w] Zp ; X_new = S[:, 0:mp] Yx + P_new (same for AS);
// W = dinv (AX_new - b X_new theta);  partial column sums of R^2 and X^2.
// M layout (T, row-major): Zp [w x mp] then Yx [mp x mp].
struct UpdArgs {
  int64_t n;
  int tk;
  int ld, w, m, mp;
  const int *skip;        // device flag: nonzero -> return (fallback iteration)
  double *part;           // [grid][2*mp]
  void *wc;               // compact W copy (n x mp), the SpMM input
};

template <typename T, int NS, int RT>
__global__ void __launch_bounds__(kFThreads, 1)
    k_update_resid(T *__restrict__ S, T *__restrict__ AS, const T *__restrict__ b,
                   const T *__restrict__ prec, const T *__restrict__ Mg,
                   const double *__restrict__ theta, UpdArgs a) {
  if (*a.skip) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int ld = a.ld, w = a.w, mp = a.mp, TK = a.tk;
  const size_t tile_elems = (size_t)TK * ld + 16;
  T *ring = reinterpret_cast<T *>(smraw);
  auto stS = [&](int s) { return ring + (size_t)s * (2 * tile_elems + TK + 16); };
  auto stA = [&](int s) { return stS(s) + tile_elems; };
  auto stB = [&](int s) { return stS(s) + 2 * tile_elems; };
  T *sM = ring + (size_t)NS * (2 * tile_elems + TK + 16);   // Zp then Yx
  const int mlen = w * mp + mp * mp;
  T *oPS = sM + mlen + 16;                                   // [TK][mp] each
  T *oPA = oPS + TK * mp;
  T *oXS = oPA + TK * mp;
  T *oXA = oXS + TK * mp;
  T *sth = oXA + TK * mp;                                    // theta (mp)
  T *sprec = sth + mp + 4;                                   // prec tile (TK)
  unsigned char *after = reinterpret_cast<unsigned char *>(sprec + TK + 4);
  after = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(after) + 15) & ~uintptr_t(15));
  uint64_t *bars = reinterpret_cast<uint64_t *>(after);
  // [kFThreads][8] column partials, used after the tile loop only: aliases
  // the (then idle) stage ring, which keeps the shared-memory budget for rows
  double *red = reinterpret_cast<double *>(smraw);

  const int tid = threadIdx.x;
  for (int e = tid; e < mlen; e += kFThreads) sM[e] = Mg[e];
  for (int e = tid; e < mp; e += kFThreads) sth[e] = e < a.m ? (T)theta[e] : T(0);
  const int64_t ntiles = (a.n + TK - 1) / TK;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_proxy_async();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < NS && t_begin + s < t_end; ++s)
      issue_tile<T>(S, AS, b, a.n, ld, TK, t_begin + s, stS(s), stA(s), stB(s), &bars[s]);

  const int R = kFThreads / mp;
  const int rc = tid % mp, rrow = tid / mp;
  double sr = 0.0, sx = 0.0;
  // fp32 residual pass: 16-byte chunks (mp % 4 == 0)
  const int C4 = mp / 4, R4 = kFThreads / (C4 > 0 ? C4 : 1);
  const int rc4 = tid % (C4 > 0 ? C4 : 1), rrow4 = tid / (C4 > 0 ? C4 : 1);
  double sr4[4] = {0.0, 0.0, 0.0, 0.0}, sx4[4] = {0.0, 0.0, 0.0, 0.0};
  const T *Zp = sM, *Yx = sM + w * mp;
  const int cb = (mp + 3) / 4, nblk = (TK / RT) * cb;  // per matrix
  for (int64_t t = t_begin; t < t_end; ++t) {
    const int s = (int)((t - t_begin) % NS);
    const uint32_t phase = (uint32_t)(((t - t_begin) / NS) & 1);
    mbar_wait(&bars[s], phase);
    const int64_t r0 = t * TK;
    const int nr = (int)min((int64_t)TK, a.n - r0);
    for (int e = tid; e < TK; e += kFThreads) sprec[e] = (e < nr && prec) ? prec[r0 + e] : T(1);
    // P_new = S Zp, then X_new = X Yx + P_new  (register blocks of RT rows x 4
    // columns; fp32 reads 4 consecutive k of each row with one 128-bit load)
    for (int phase = 0; phase < 2; ++phase) {
      const int K = phase == 0 ? w : mp;
      const T *Bm = phase == 0 ? Zp : Yx;
      // a job owns RT rows rb, rb + RS, rb + 2 RS, ... (RS = TK / RT): with
      // the odd 16-byte row stride, 8 consecutive rb hit distinct bank groups
      // Jobs are grouped so a warp reads at most 8 distinct 16-byte B chunks
      // (one shared-memory wavefront): column blocks 0-7 first, then 8+.
      const int RS = TK / RT;
      const int nrb = TK / RT, cbA = min(cb, 8), cbB = cb - cbA;
      const int nJA = 2 * nrb * cbA;
      for (int job = tid; job < 2 * nblk; job += kFThreads) {
        int mat, rb, c0;
        if (job < nJA) {
          mat = job / (nrb * cbA);
          const int rem = job - mat * nrb * cbA;
          rb = rem / cbA;
          c0 = (rem - rb * cbA) * 4;
        } else {
          const int j2 = job - nJA;
          mat = j2 / (nrb * cbB);
          const int rem = j2 - mat * nrb * cbB;
          rb = rem / cbB;
          c0 = (8 + rem - rb * cbB) * 4;
        }
        const T *src = (mat ? stA(s) : stS(s)) + rb * ld;
        T acc[RT][4];
        if (phase == 0) {
#pragma unroll
          for (int x = 0; x < RT; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = T(0);
        } else {
          const T *pn = (mat ? oPA : oPS) + rb * mp + c0;
          if constexpr (sizeof(T) == 4) {  // mp % 4 == 0 for fp32
#pragma unroll
            for (int x = 0; x < RT; ++x) {
              const float4 v = *reinterpret_cast<const float4 *>(pn + x * RS * mp);
              acc[x][0] = v.x;
              acc[x][1] = v.y;
              acc[x][2] = v.z;
              acc[x][3] = v.w;
            }
          } else {
#pragma unroll
            for (int x = 0; x < RT; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[x][y] = (c0 + y < mp) ? pn[x * RS * mp + y] : T(0);
          }
        }
        if constexpr (sizeof(T) == 4) {
#pragma unroll 3
          for (int k = 0; k < K; k += 4) {
            float4 b[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              b[kk] = *reinterpret_cast<const float4 *>(Bm + (k + kk) * mp + c0);
#pragma unroll
            for (int x = 0; x < RT; ++x) {
              const float4 av = *reinterpret_cast<const float4 *>(src + x * RS * ld + k);
              const float aa[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                acc[x][0] += aa[kk] * b[kk].x;
                acc[x][1] += aa[kk] * b[kk].y;
                acc[x][2] += aa[kk] * b[kk].z;
                acc[x][3] += aa[kk] * b[kk].w;
              }
            }
          }
        } else {
          for (int k = 0; k < K; ++k) {
            T mz[4];
#pragma unroll
            for (int y = 0; y < 4; ++y) mz[y] = Bm[k * mp + c0 + y];
#pragma unroll
            for (int x = 0; x < RT; ++x) {
              const T u = src[x * RS * ld + k];
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[x][y] += u * mz[y];
            }
          }
        }
        T *dst = (phase == 0 ? (mat ? oPA : oPS) : (mat ? oXA : oXS)) + rb * mp + c0;
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int x = 0; x < RT; ++x)
            *reinterpret_cast<float4 *>(dst + x * RS * mp) =
                make_float4(acc[x][0], acc[x][1], acc[x][2], acc[x][3]);
        } else {
#pragma unroll
          for (int x = 0; x < RT; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y)
              if (c0 + y < mp) dst[x * RS * mp + y] = acc[x][y];
        }
      }
      __syncthreads();
    }
    // residual + W, and write back [X P W] / [AX AP] rows
    if constexpr (sizeof(T) == 4) {
      // one 16-byte column chunk per thread (fixed chunk: rows rr4, rr4 + R4, ...)
      for (int rr = rrow4; rr < nr && rrow4 < R4; rr += R4) {
        const float4 x = *reinterpret_cast<const float4 *>(oXS + rr * mp + 4 * rc4);
        const float4 ax = *reinterpret_cast<const float4 *>(oXA + rr * mp + 4 * rc4);
        const float xs[4] = {x.x, x.y, x.z, x.w}, axs[4] = {ax.x, ax.y, ax.z, ax.w};
        const float br = stB(s)[rr], pr = sprec[rr];
        float wv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wv[q] = 0.f;
          if (4 * rc4 + q < a.m) {
            const float r = axs[q] - br * xs[q] * sth[4 * rc4 + q];
            sr4[q] += (double)r * (double)r;
            sx4[q] += (double)xs[q] * (double)xs[q];
            wv[q] = pr * r;
          }
        }
        const float4 w4 = make_float4(wv[0], wv[1], wv[2], wv[3]);
        float *srow = S + (r0 + rr) * ld + 4 * rc4;
        float *arow = AS + (r0 + rr) * ld + 4 * rc4;
        *reinterpret_cast<float4 *>(srow) = x;
        *reinterpret_cast<float4 *>(srow + mp) =
            *reinterpret_cast<const float4 *>(oPS + rr * mp + 4 * rc4);
        *reinterpret_cast<float4 *>(srow + 2 * mp) = w4;
        reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.wc) + (r0 + rr) * mp)[rc4] = w4;
        *reinterpret_cast<float4 *>(arow) = ax;
        *reinterpret_cast<float4 *>(arow + mp) =
            *reinterpret_cast<const float4 *>(oPA + rr * mp + 4 * rc4);
      }
    } else {
      for (int rr = rrow; rr < nr && rrow < R; rr += R) {
        const T x = oXS[rr * mp + rc];
        const T ax = oXA[rr * mp + rc];
        T wv = T(0);
        if (rc < a.m) {
          const T bx = stB(s)[rr] * x;
          const T r = ax - bx * sth[rc];
          sr += (double)r * (double)r;
          sx += (double)x * (double)x;
          wv = sprec[rr] * r;
        }
        T *srow = S + (r0 + rr) * ld;
        T *arow = AS + (r0 + rr) * ld;
        srow[rc] = x;
        srow[mp + rc] = oPS[rr * mp + rc];
        srow[2 * mp + rc] = wv;
        reinterpret_cast<T *>(a.wc)[(r0 + rr) * mp + rc] = wv;
        arow[rc] = ax;
        arow[mp + rc] = oPA[rr * mp + rc];
      }
    }
    __syncthreads();  // stage s and the output tiles are free
    if (tid == 0 && t + NS < t_end) {
      fence_proxy_async();
      issue_tile<T>(S, AS, b, a.n, ld, TK, t + NS, stS(s), stA(s), stB(s), &bars[s]);
    }
  }
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[tid * 8 + q] = (rrow4 < R4) ? sr4[q] : 0.0;
      red[tid * 8 + 4 + q] = (rrow4 < R4) ? sx4[q] : 0.0;
    }
    __syncthreads();
    for (int c = tid; c < 2 * mp; c += kFThreads) {
      const int col = c % mp, which = c / mp;
      double s2 = 0.0;
      for (int q = 0; q < R4; ++q) s2 += red[(q * C4 + col / 4) * 8 + 4 * which + (col & 3)];
      a.part[(size_t)blockIdx.x * 2 * mp + c] = s2;
    }
  } else {
    red[tid * 2] = (rrow < R) ? sr : 0.0;
    red[tid * 2 + 1] = (rrow < R) ? sx : 0.0;
    __syncthreads();
    for (int c = tid; c < 2 * mp; c += kFThreads) {
      const int col = c % mp, which = c / mp;
      double s2 = 0.0;
      for (int q = 0; q < R; ++q) s2 += red[(q * mp + col) * 2 + which];
      a.part[(size_t)blockIdx.x * 2 * mp + c] = s2;
    }
  }
}

// ------------------------------------------------------------ k_update_ws ---
// fp32 k_update_resid with warp specialisation: warps 0-7 form the P / X
// register-blocked products of tile t while warps 8-11 run the residual, W,
// column norms and the global write-back of tile t-1 (double-buffered output
// tiles).  In k_update_resid those phases alternate behind __syncthreads and
// the FMA pipes idle during the write-back (~30 % of the samples, ncu).
// Barriers: full[s] (TMA), rdy[o] (8 FMA warps -> output tile o complete),
// fre[o] (4 store warps -> output tile o consumed, stage refilled).
constexpr int kWsF = 256, kWsS = 128;
#ifndef MG_WS_NS
#define MG_WS_NS 2
#endif
constexpr int kWsNS = MG_WS_NS;  // TMA ring stages (one tile of look-ahead covers the latency)

__device__ __forceinline__ void mbar_arrive_cta(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__host__ __device__ inline size_t upd_ws_bytes(int tk, int ld, int w, int mp) {
  const size_t tile = (size_t)tk * ld + 16;
  return (size_t)kWsNS * (2 * tile + tk + 16) * 4 + ((size_t)w * mp + (size_t)mp * mp + 16) * 4 +
         (size_t)8 * tk * mp * 4 + (size_t)(mp + 4) * 4 + 256;
}

template <int RT>
__global__ void __launch_bounds__(kWsF + kWsS, 1)
    k_update_ws(float *__restrict__ S, float *__restrict__ AS, const float *__restrict__ b,
                const float *__restrict__ prec, const float *__restrict__ Mg,
                const double *__restrict__ theta, UpdArgs a) {
  if (*a.skip) return;
  constexpr int NS = kWsNS;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int ld = a.ld, w = a.w, mp = a.mp, TK = a.tk;
  const size_t tile_elems = (size_t)TK * ld + 16;
  float *ring = reinterpret_cast<float *>(smraw);
  auto stS = [&](int s) { return ring + (size_t)s * (2 * tile_elems + TK + 16); };
  auto stA = [&](int s) { return stS(s) + tile_elems; };
  auto stB = [&](int s) { return stS(s) + 2 * tile_elems; };
  float *sM = ring + (size_t)NS * (2 * tile_elems + TK + 16);
  const int mlen = w * mp + mp * mp;
  float *obuf = sM + mlen + 16;  // [2][4][TK][mp]: P_S, P_A, X_S, X_A
  auto oP = [&](int o, int mat) { return obuf + ((size_t)o * 4 + mat) * TK * mp; };
  auto oX = [&](int o, int mat) { return obuf + ((size_t)o * 4 + 2 + mat) * TK * mp; };
  float *sth = obuf + (size_t)8 * TK * mp;
  unsigned char *after = reinterpret_cast<unsigned char *>(sth + mp + 4);
  after = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(after) + 15) & ~uintptr_t(15));
  uint64_t *full = reinterpret_cast<uint64_t *>(after);
  uint64_t *rdy = full + NS, *fre = rdy + 2;
  double *red = reinterpret_cast<double *>(smraw);  // after the loop (aliases the ring)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < mlen; e += blockDim.x) sM[e] = Mg[e];
  for (int e = tid; e < mp; e += blockDim.x) sth[e] = e < a.m ? (float)theta[e] : 0.f;
  const int64_t ntiles = (a.n + TK - 1) / TK;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) mbar_init(&full[q], 1);
    for (int q = 0; q < 2; ++q) {
      mbar_init(&rdy[q], kWsF / 32);
      mbar_init(&fre[q], kWsS / 32);
    }
    fence_proxy_async();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < NS && t_begin + q < t_end; ++q)
      issue_tile<float>(S, AS, b, a.n, ld, TK, t_begin + q, stS(q), stA(q), stB(q), &full[q]);

  const int C4 = mp / 4, R4 = kWsS / C4;
  double sr4[4] = {0.0, 0.0, 0.0, 0.0}, sx4[4] = {0.0, 0.0, 0.0, 0.0};
  if (tid < kWsF) {
    // ------------------------------------------------------ FMA warps
    const float *Zp = sM, *Yx = sM + w * mp;
    const int cb = (mp + 3) / 4, nblk = (TK / RT) * cb;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int lt = (int)(t - t_begin), s = lt % NS, o = lt & 1;
      mbar_wait(&full[s], (uint32_t)((lt / NS) & 1));
      mbar_wait(&fre[o], (uint32_t)(((lt >> 1) & 1) ^ 1));
      for (int phase = 0; phase < 2; ++phase) {
        const int K = phase == 0 ? w : mp;
        const float *Bm = phase == 0 ? Zp : Yx;
        const int RS = TK / RT;
        const int nrb = TK / RT, cbA = min(cb, 8), cbB = cb - cbA;
        const int nJA = 2 * nrb * cbA;
        for (int job = tid; job < 2 * nblk; job += kWsF) {
          int mat, rb, c0;
          if (job < nJA) {
            mat = job / (nrb * cbA);
            const int rem = job - mat * nrb * cbA;
            rb = rem / cbA;
            c0 = (rem - rb * cbA) * 4;
          } else {
            const int j2 = job - nJA;
            mat = j2 / (nrb * cbB);
            const int rem = j2 - mat * nrb * cbB;
            rb = rem / cbB;
            c0 = (8 + rem - rb * cbB) * 4;
          }
          const float *src = (mat ? stA(s) : stS(s)) + rb * ld;
          float acc[RT][4];
          if (phase == 0) {
#pragma unroll
            for (int x = 0; x < RT; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
          } else {
            const float *pn = oP(o, mat) + rb * mp + c0;
#pragma unroll
            for (int x = 0; x < RT; ++x) {
              const float4 v = *reinterpret_cast<const float4 *>(pn + x * RS * mp);
              acc[x][0] = v.x;
              acc[x][1] = v.y;
              acc[x][2] = v.z;
              acc[x][3] = v.w;
            }
          }
          // register double buffering: the next k-quad's shared-memory loads
          // are in flight while this quad's FMAs issue (short-scoreboard stalls
          // on LDS dominated the FMA phase)
          float4 bb[4], av[RT];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) bb[kk] = *reinterpret_cast<const float4 *>(Bm + kk * mp + c0);
#pragma unroll
          for (int x = 0; x < RT; ++x) av[x] = *reinterpret_cast<const float4 *>(src + x * RS * ld);
#pragma unroll 2
          for (int k = 0; k < K; k += 4) {
            float4 nb[4], na[RT];
            const int kn = k + 4 < K ? k + 4 : k;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              nb[kk] = *reinterpret_cast<const float4 *>(Bm + (kn + kk) * mp + c0);
#pragma unroll
            for (int x = 0; x < RT; ++x)
              na[x] = *reinterpret_cast<const float4 *>(src + x * RS * ld + kn);
#pragma unroll
            for (int x = 0; x < RT; ++x) {
              const float aa[4] = {av[x].x, av[x].y, av[x].z, av[x].w};
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                acc[x][0] += aa[kk] * bb[kk].x;
                acc[x][1] += aa[kk] * bb[kk].y;
                acc[x][2] += aa[kk] * bb[kk].z;
                acc[x][3] += aa[kk] * bb[kk].w;
              }
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) bb[kk] = nb[kk];
#pragma unroll
            for (int x = 0; x < RT; ++x) av[x] = na[x];
          }
          float *dst = (phase == 0 ? oP(o, mat) : oX(o, mat)) + rb * mp + c0;
#pragma unroll
          for (int x = 0; x < RT; ++x)
            *reinterpret_cast<float4 *>(dst + x * RS * mp) =
                make_float4(acc[x][0], acc[x][1], acc[x][2], acc[x][3]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kWsF) : "memory");  // FMA warps only
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&rdy[o]);  // release: tile o's products visible
    }
  } else {
    // ---------------------------------------------------- store warps
    const int st = tid - kWsF;
    const int rc4 = st % C4, rrow4 = st / C4;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int lt = (int)(t - t_begin), s = lt % NS, o = lt & 1;
      mbar_wait(&rdy[o], (uint32_t)((lt >> 1) & 1));
      const int64_t r0 = t * TK;
      const int nr = (int)min((int64_t)TK, a.n - r0);
      for (int rr = rrow4; rr < nr && rrow4 < R4; rr += R4) {
        const float4 x = *reinterpret_cast<const float4 *>(oX(o, 0) + rr * mp + 4 * rc4);
        const float4 ax = *reinterpret_cast<const float4 *>(oX(o, 1) + rr * mp + 4 * rc4);
        const float xs[4] = {x.x, x.y, x.z, x.w}, axs[4] = {ax.x, ax.y, ax.z, ax.w};
        const float br = stB(s)[rr], pr = prec ? prec[r0 + rr] : 1.f;
        float wv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wv[q] = 0.f;
          if (4 * rc4 + q < a.m) {
            const float r = axs[q] - br * xs[q] * sth[4 * rc4 + q];
            sr4[q] += (double)r * (double)r;
            sx4[q] += (double)xs[q] * (double)xs[q];
            wv[q] = pr * r;
          }
        }
        const float4 w4 = make_float4(wv[0], wv[1], wv[2], wv[3]);
        float *srow = S + (r0 + rr) * ld + 4 * rc4;
        float *arow = AS + (r0 + rr) * ld + 4 * rc4;
        *reinterpret_cast<float4 *>(srow) = x;
        *reinterpret_cast<float4 *>(srow + mp) =
            *reinterpret_cast<const float4 *>(oP(o, 0) + rr * mp + 4 * rc4);
        *reinterpret_cast<float4 *>(srow + 2 * mp) = w4;
        reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.wc) + (r0 + rr) * mp)[rc4] = w4;
        *reinterpret_cast<float4 *>(arow) = ax;
        *reinterpret_cast<float4 *>(arow + mp) =
            *reinterpret_cast<const float4 *>(oP(o, 1) + rr * mp + 4 * rc4);
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kWsS) : "memory");  // store warps only
      if (st == 0 && t + NS < t_end) {  // stage s fully consumed: refill it
        fence_proxy_async();
        issue_tile<float>(S, AS, b, a.n, ld, TK, t + NS, stS(s), stA(s), stB(s), &full[s]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&fre[o]);
    }
  }
  __syncthreads();
  if (tid >= kWsF) {
    const int st = tid - kWsF;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[st * 8 + q] = (st / C4 < R4) ? sr4[q] : 0.0;
      red[st * 8 + 4 + q] = (st / C4 < R4) ? sx4[q] : 0.0;
    }
  }
  __syncthreads();
  for (int c = tid; c < 2 * mp; c += blockDim.x) {
    const int col = c % mp, which = c / mp;
    double s2 = 0.0;
    for (int q = 0; q < R4; ++q) s2 += red[(q * C4 + col / 4) * 8 + 4 * which + (col & 3)];
    a.part[(size_t)blockIdx.x * 2 * mp + c] = s2;
  }
}

// C[i][j] = sum_u A(i, u) B(u, j), A(i, u) = A[i*ai + u*au], B(u, j) = B[u*bu + j],
// i < R, j < Cn, ascending u (the same fma chain per entry as a scalar loop),
// 4x4 register tiles per thread: 8 shared loads per 16 fma instead of 2 per 1
// (the scalar loops were ~20 % of k_ctrl_fast at m = 33)
__device__ inline void blk_gemm4(const double *__restrict__ A, int ai, int au,
                                 const double *__restrict__ B, int bu, double *__restrict__ C,
                                 int ldc, int R, int Cn, int K) {
  const int tr = (R + 3) / 4, tc = (Cn + 3) / 4;
  for (int t = threadIdx.x; t < tr * tc; t += blockDim.x) {
    const int i0 = (t / tc) * 4, j0 = (t % tc) * 4;
    int ii[4], jj[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      ii[x] = min(i0 + x, R - 1) * ai;
      jj[x] = min(j0 + x, Cn - 1);
    }
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
    for (int u = 0; u < K; ++u) {
      double av[4], bv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) av[x] = A[ii[x] + u * au];
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = B[u * bu + jj[y]];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y)
        if (i0 + x < R && j0 + y < Cn) C[(i0 + x) * ldc + j0 + y] = acc[x][y];
  }
}

// ---------------------------------------------------------- k_ctrl_fast ---
// Small-matrix LOBPCG step for a prefix iteration.  G_B / G_A are w x w over
// physical columns [0, w) = [X | P | W].  Logical basis: X (m trusted
// columns), then V = (active W, valid P) in the reference's order.
//   X~ = X RX^-1 with RX = chol(G_XX)       (X re-orthonormalised every step)
//   C  = X~'BV, D = RX^-1 C                 (projection, eigensolver.py:126-129)
//   Gv = G_VV - C'C                         (B-Gram of V - X~ C)
//   Cholesky with the drop rule on Gv       (eigensolver.py:133-152)
//   T  = [[I, -D Rinv], [0, Rinv]];  G_RR = T' G_A T;  eigh (Jacobi)
// Fallback flag when any kept column's pivot^2 < fast_tol * (its un-projected
// B-norm^2): the multi-pass path then materialises the projections instead.
struct FastArgs {
  int m, mp, w;
  int nv;
  int vcols[kMaxFast];    // physical columns of V in logical order
  double fast_tol;
  double rel_tol, abs_tol;
  int use_global;
  int clk_off;            // >0: write phase clocks at scratch[clk_off...] (debug)
};

template <typename T>
__global__ void __launch_bounds__(512)
    k_ctrl_fast(FastArgs a, const double *__restrict__ GB, const double *__restrict__ GA,
                T *__restrict__ Mout, double *__restrict__ theta, int *status, double *scratch) {
  extern __shared__ __align__(16) double smf[];
  __shared__ int keep[kMaxFast];
  __shared__ int rank[kMaxFast];
  __shared__ double wv[kMaxFast];
  __shared__ double orig[kMaxFast];
  __shared__ double unproj[kMaxFast];
  __shared__ double red[512];
  __shared__ double red2[512];
  __shared__ double et[kMaxFast], ed[kMaxFast], ee[kMaxFast], elo[kMaxFast], ehi[kMaxFast];
  __shared__ int ecnt[512];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int m = a.m, nv = a.nv, w = a.w, mp = a.mp;
  long long *tclk = reinterpret_cast<long long *>(scratch + a.clk_off);
  int tph = 0;
#define MG_TICK() \
  do {              \
    if (a.clk_off > 0 && tid == 0) tclk[tph++] = clock64(); \
  } while (0)
  MG_TICK();
  // global scratch: C, D [m x nv]; RX, RXi [m x m]; T, HT [w x smax]
  double *C = scratch;
  double *D = C + m * nv;
  double *RX = D + m * nv;
  double *RXi = RX + m * m;
  double *GX = RXi + m * m;
  const int smax = m + nv;
  double *Tm = GX + m * m;
  double *HT = Tm + (size_t)w * smax;
  double *big = HT + (size_t)w * smax;
  double *Gv = a.use_global ? big : smf;
  double *R = Gv + nv * nv;
  if (tid == 0) bad = 0;
  // X is re-orthonormalised from its own B-Gram every step (X~ = X RX^-1), so
  // single-pass rounding in the previous update never accumulates
  for (int e = tid; e < m * m; e += nt) GX[e] = GB[(e / m) * w + (e % m)];
  __syncthreads();
  const int nkx = blk_cholesky_drop(GX, m, m, 0.0, RX, m, keep, orig, 1e-6, 1e-300);
  if (nkx < m) {
    if (tid == 0) status[5] = 1;
    return;
  }
  blk_tri_inv_kept(RX, m, m, keep, RXi, m);
  MG_TICK();
  for (int e = tid; e < m * nv; e += nt) {  // C = RX^-T G_XV
    int x = e / nv, q = e - x * nv;
    double s2 = 0.0;
    for (int y = 0; y <= x; ++y) s2 += RXi[y * m + x] * GB[y * w + a.vcols[q]];
    C[e] = s2;
  }
  __syncthreads();
  for (int e = tid; e < m * nv; e += nt) {  // D = RX^-1 C  (X coefficients of the projection)
    int x = e / nv, q = e - x * nv;
    double s2 = 0.0;
    for (int y = x; y < m; ++y) s2 += RXi[x * m + y] * C[y * nv + q];
    D[e] = s2;
  }
  for (int e = tid; e < nv * nv; e += nt) {  // Gv = G_VV - C'C
    int p = e / nv, q = e - p * nv;
    double s2 = GB[a.vcols[p] * w + a.vcols[q]];
    for (int x = 0; x < m; ++x) s2 -= C[x * nv + p] * C[x * nv + q];
    Gv[e] = s2;
    if (p == q) unproj[p] = GB[a.vcols[p] * w + a.vcols[p]];
  }
  __syncthreads();
  MG_TICK();
  blk_check_finite(Gv, nv, nv, nv, status + 4, 16);
  const int nk = blk_cholesky_drop(Gv, nv, nv, 1.0, R, nv, keep, orig, a.rel_tol, a.abs_tol);
  // quality: every kept pivot must be resolvable from the Gram at this precision
  for (int q = tid; q < nv; q += nt)
    if (keep[q]) {
      double piv = R[q * nv + q];
      if (!(piv * piv >= a.fast_tol * unproj[q])) atomicOr(&bad, 1);
    }
  __syncthreads();
  if (bad) {
    if (tid == 0) status[5] = 1;
    return;
  }
  MG_TICK();
  blk_tri_inv_kept(R, nv, nv, keep, Gv, nv);  // Gv <- Rinv
  MG_TICK();
  if (tid == 0) {
    int r = 0;
    for (int t = 0; t < nv; ++t) rank[t] = keep[t] ? r++ : -1;
  }
  __syncthreads();
  const int s = m + nk;
  for (int e = tid; e < w * s; e += nt) Tm[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) Tm[(e / m) * s + (e % m)] = RXi[e];
  for (int e = tid; e < nv * nv; e += nt) {
    int p = e / nv, t = e - p * nv;
    if (keep[t] && keep[p] && p <= t) Tm[a.vcols[p] * s + m + rank[t]] = Gv[p * nv + t];
  }
  for (int e = tid; e < m * nv; e += nt) {  // X rows: -D Rinv
    int x = e / nv, t = e - x * nv;
    if (!keep[t]) continue;
    double s2 = 0.0;
    for (int p = 0; p <= t; ++p)
      if (keep[p]) s2 += D[x * nv + p] * Gv[p * nv + t];
    Tm[x * s + m + rank[t]] = -s2;
  }
  __syncthreads();
  MG_TICK();
  blk_gemm4(GA, w, 1, Tm, s, HT, s, w, s, w);  // HT = G_A T
  __syncthreads();
  double *Aj = a.use_global ? big + 2 * nv * nv : smf;
  double *Vj = Aj + s * s;
  blk_gemm4(Tm, 1, s, HT, s, Aj, s, s, s, w);  // Aj = T' HT
  __syncthreads();
  for (int e = tid; e < s * s; e += nt) {
    int i = e / s, j = e - i * s;
    if (i < j) {
      double v = 0.5 * (Aj[i * s + j] + Aj[j * s + i]);
      Aj[i * s + j] = v;
      Aj[j * s + i] = v;
    }
  }
  __syncthreads();
  MG_TICK();
  blk_check_finite(Aj, s, s, s, status + 4, 8);
  const int take = min(m, s);
  {
    double *lu = big + 2 * nv * nv + 2 * (size_t)smax * smax;  // dedicated LU scratch
    EigWork ew{et, ed, ee, elo, ehi, ecnt, red, red2, lu};
    if (a.clk_off > 0) ew.clk = tclk + 20;
    blk_eig_smallest(Aj, s, s, take, wv, Vj, take, ew);
  }
  MG_TICK();
  for (int i = tid; i < take; i += nt) theta[i] = wv[i];
  // Zp [w x mp] = T[:, m:s] Y[m:s, :take];  Yx [mp x mp] = RX^-1 Y[0:m, :take]
  for (int e = tid; e < w * mp; e += nt) {
    int r = e / mp, c = e - r * mp;
    double s2 = 0.0;
    if (c < take)
      for (int u = m; u < s; ++u) s2 += Tm[r * s + u] * Vj[u * take + c];
    Mout[e] = (T)s2;
  }
  for (int e = tid; e < mp * mp; e += nt) {
    int x = e / mp, c = e - x * mp;
    double v = 0.0;
    if (x < m && c < take)
      for (int y = x; y < m; ++y) v += RXi[x * m + y] * Vj[y * take + c];
    Mout[w * mp + e] = (T)v;
  }
  __syncthreads();
  MG_TICK();
  if (tid == 0) {
    status[0] = nk;
    status[1] = take;
    status[2] = nk;
    status[3] = s;
    status[5] = 0;
  }
#undef MG_TICK
}

}  // namespace mg
