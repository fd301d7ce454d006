// tcgen05 Gram pair, TMA-fed (v2): G_B = S' diag(b) S and G_A = S' (AS) for
// the fp32 fast path at wide blocks (w = 3mp in (64, 128]).
//
// Why a second kernel (profiles/r1_ncu_c5_2M.md): v1 (mg_tc.cu) permutes every
// element of S / AS into a no-swizzle K-major operand with the worker warps,
// and both CTAs of a pair convert the whole 'A' side -- the converters, not
// the tensor pipe (20 % active) or HBM (16 %), set its pace.
//
// v2 lets the tensor core read the tiles almost as they arrive:
//   * each row tile of S and AS is loaded by TMA (cp.async.bulk.tensor.2d,
//     SWIZZLE_128B_ATOM_32B, 32-column panels): that IS the canonical
//     MN-major tf32 operand layout (SWIZZLE_128B_BASE32B; M / N = the Gram
//     index = S column, contiguous; K = tile rows), so no layout permutation;
//   * the worker warps only do element-wise work: hi = rn_tf32(x) in place,
//     lo = x - hi, bS = b_r x and its pieces (round-to-nearest hi keeps the
//     products unbiased: with the hardware's truncation as hi, long positive
//     sums such as diag(G_B) drift by ~2^-22 relative);
//   * 2 MMAs per k-step: A_hi x [B_hi | B_lo] (hi*hi and hi*lo side by side,
//     N = 64 pw) and A_lo x B_hi into the cross columns;
//   * short TMEM accumulations (128 rows, double-buffered) drained into fp32
//     registers, folded into fp64 every 2048 rows (the TC's fp32 adds are not
//     round-to-nearest: 2048-row TMEM sums failed the 2e-6 bar).
// Measured (profiles/r1_gram_tc.md): 11-13 ms at 20M x 108 vs 16.8 ms (v1);
// the per-tile pipeline (~0.5 us per 16-row tile even with the MMAs and the
// element-wise work disabled) bounds it, not HBM or the tensor pipe.
// Mirror convention (as v1 / k_reduce_gram2): entries of block-lower 8x8
// blocks come from the block-upper product, so only j >= 8 floor(i/8) is
// drained.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "mg_fastk.cuh"
#include "mg_tc.cuh"

namespace mg {

namespace {

constexpr int kG2Threads = 320;   // warp 0 TMA producer, warp 1 MMA issuer, 8 worker warps
constexpr int kG2TK = 32;         // rows per stage (4 MMA k-steps)
constexpr int kG2Stages = 3;
constexpr int kG2Panel = kG2TK * 128;  // bytes per 32-column panel of a stage
constexpr int kG2FL = 4;          // tiles per TMEM accumulation group (128 rows)
constexpr int kG2FoldG = 16;      // groups per fp64 fold (2048 rows)

__host__ __device__ constexpr size_t g2_smem_bytes(int pw) {
  return kG2Stages * ((size_t)4 * pw * kG2Panel + 128) + 256;
}

// Shared-memory descriptor (sm_100 version 1) of an MN-major tf32 operand in
// the SWIZZLE_128B_BASE32B layout -- the only MN-major smem layout tf32 has
// (32-byte granules of each 128-byte row XOR-ed with the row index mod 4; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes it).  LBO = stride between
// 32-column panels (MN direction), SBO = stride between 4-row groups (K).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
// D f32, A/B tf32, both operands MN-major
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tcf_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tcf_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *map, int c0, int r0,
                                       uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_3d(void *dst, const CUtensorMap *map, int r0, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_1d(void *dst, const CUtensorMap *map, int c0, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2}], [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16_pair(uint32_t ta, uint32_t tb, float *va, float *vb) {
  uint32_t r[32];
#define MG_R8(o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), \
                 "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7])
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : MG_R8(0), MG_R8(8)
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : MG_R8(16), MG_R8(24)
      : "r"(tb));
#undef MG_R8
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    va[q] = __uint_as_float(r[q]);
    vb[q] = __uint_as_float(r[16 + q]);
  }
}
__device__ __forceinline__ float trunc_tf32(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// round to nearest (ties away) TF32, integer ops
__device__ __forceinline__ float rn_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// x = hi + lo: hi = rn_tf32(x) (unbiased), lo = x - hi exact in fp32 (the
// MMA truncates it; error <= 2^-23 |x|)
__device__ __forceinline__ void split4(float4 x, float4 &hi, float4 &lo) {
  hi = make_float4(rn_tf32(x.x), rn_tf32(x.y), rn_tf32(x.z), rn_tf32(x.w));
  lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
}

// drain TMEM group fg (this thread: lane-quadrant row i, column half ch) into
// the fp32 register accumulators; fold them into fp64 every kG2FoldG groups
__device__ __forceinline__ void g2_drain(int fg, int NG, uint64_t *tmf, uint64_t *tme,
                                         uint32_t tbase, int q, int ch, int hw, int lane, int i,
                                         int jmin, int w, double *dp, float (&acc)[64],
                                         bool skip, bool full, int wneed) {
  const int buf = fg & 1;
  mbar_wait(&tmf[buf], (fg >> 1) & 1);
  __syncwarp();
  tcf_after();
  const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + buf * 256 + ch * hw;
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    // warp-uniform: block-lower chunks are skipped (mirror convention); in the
    // narrow mode (full) only B columns 8 .. 43 of each 64-column half are W columns
    if (!skip && c < hw && (full ? c < wneed : ch * hw + c + 16 > 32 * q)) {
      float v[16], x[16];
      tmem_ld16_pair(ta + c, ta + 32 * (hw / 16) + c, v, x);
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[c + e] += v[e] + x[e];
    }
  }
  tcf_before();
  __syncwarp();
  if (lane == 0) arrive(&tme[buf]);
  if ((fg + 1) % kG2FoldG == 0 || fg == NG - 1) {
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const int j = ch * hw + c;
      if (c < hw && j >= jmin && (full || j < w) && i < w) dp[(size_t)j * 128 + i] += (double)acc[c];
      acc[c] = 0.f;
    }
  }
}

struct Gram2TcArgs {
  int64_t n;
  int w, pw;      // Gram width, 32-column panels (w <= 32 pw, pw in 2..4)
  int pwf;        // full panels (w / 32), loaded by the 3-D maps
  int npairs;     // grid = 2 * npairs
  int dbg;        // MG_TC2_DBG timing experiments: 1 no MMA, 2 no derive, 4 no drain
  int narrow;     // 1: W-column blocks only: every CTA owns a row range and forms
                  // S' [bS(:, 32 pw0:) | AS(:, 32 pw0:)] with pw0 = pw / 2 (the panels that
                  // hold W: pw = 4, mp = 36: columns [72, 108) in panels 2-3; pw = 2,
                  // mp = 20: columns [40, 60) in panel 1)
  int wneed;      // narrow: B columns of each half that are drained (multiple of 16)
  double *part;   // [pair][h][128 (j)][128 (i)] fp64, zeroed by the host
};

// CTA pair (2c, 2c+1) owns a contiguous row range; CTA 2c+h computes G_h
// (h = 0: G_B, A = S, B = bS; h = 1: G_A, A = S, B = AS) over ALL its rows.
// Stage layout (pw panels of kG2Panel bytes, 1024-aligned):
//   A_hi (TMA S, rounded in place) | A_lo | B_hi (bS, or TMA AS rounded in
//   place) | B_lo
// TMEM: 2 accumulation buffers x [hi*hi (32 pw columns) | cross (32 pw)]; a buffer
// collects kG2FL tiles (128 rows) and is drained into fp32 registers while
// the other fills -- short tensor-core accumulations keep its fp32 adds'
// rounding at the v1 level; registers fold into fp64 every kG2FoldG groups.
__global__ void __launch_bounds__(kG2Threads, 1)
    k_gram_tc2(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmA,
               const __grid_constant__ CUtensorMap tmS3, const __grid_constant__ CUtensorMap tmA3,
               const __grid_constant__ CUtensorMap tmB, Gram2TcArgs a) {
  // the dynamic window starts 1024-aligned (no static shared memory here);
  // keeping the __shared__ array itself as the base lets the compiler emit
  // LDS/STS rather than generic loads
  extern __shared__ __align__(1024) unsigned char sm[];
  const int pw = a.pw;
  const uint32_t PB = (uint32_t)pw * kG2Panel;  // bytes of one pw-panel group
  const size_t SB = 4 * (size_t)PB;
  // b tiles: one 128-byte slot per stage (TMA destinations are 128-byte aligned)
  float *sb = reinterpret_cast<float *>(sm + kG2Stages * SB);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sb + kG2Stages * 32);
  uint64_t *full = bars, *drv = bars + kG2Stages, *empty = bars + 2 * kG2Stages;
  uint64_t *tmf = bars + 3 * kG2Stages, *tme = tmf + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tme + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool narrow = a.narrow != 0;
  const int h = narrow ? 1 : (blockIdx.x & 1), pair = narrow ? blockIdx.x : (blockIdx.x >> 1);
  const int64_t ntiles = (a.n + kG2TK - 1) / kG2TK;
  const int64_t t0 = ntiles * pair / a.npairs, t1 = ntiles * (pair + 1) / a.npairs;
  const int T = (int)(t1 - t0);
  const int NG = (T + kG2FL - 1) / kG2FL;  // TMEM accumulation groups

  if (tid == 0) {
    for (int s = 0; s < kG2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&drv[s], 8);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmf[s], 1);
      mbar_init(&tme[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tcf_before();
  __syncthreads();
  tcf_after();
  const uint32_t tbase = *tslot;
  if ((smem_u32(sm) & 1023) != 0) __trap();  // SW128 operand atoms need 1024-byte alignment

  if (warp == 0) {
    // --------------------------------------------------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmS)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmS3)) : "memory");
      if (h) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA3)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(
                       reinterpret_cast<uint64_t>(h ? &tmA : &tmB)) : "memory");
      if (narrow) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      for (int t = 0; t < T; ++t) {
        const int s = t % kG2Stages;
        mbar_wait(&empty[s], ((t / kG2Stages) & 1) ^ 1);
        unsigned char *st = sm + s * SB;
        mbar_expect_tx(&full[s], narrow ? PB + (pw - pw / 2) * kG2Panel + kG2TK * 4
                                        : (h ? 2 * PB : PB + kG2TK * 4));
        const int r0 = (int)((t0 + t) * kG2TK);
        if (!h || narrow) tma_1d(sb + s * 32, &tmB, r0, &full[s]);
        if (narrow) {
          // S: all panels (A side); AS: the panels that hold the W block
          if (a.pwf) tma_3d(st, &tmS3, r0, &full[s]);
          for (int p = a.pwf; p < pw; ++p) tma_2d(st + p * kG2Panel, &tmS, 32 * p, r0, &full[s]);
          for (int p = pw / 2; p < pw; ++p)
            tma_2d(st + 2 * PB + p * kG2Panel, &tmA, 32 * p, r0, &full[s]);
          continue;
        }
        // full 32-column panels in one 3-D box, the partial last panel (zero
        // beyond w) as a 2-D box: 2 TMA instructions per matrix and tile
        if (a.pwf) {
          tma_3d(st, &tmS3, r0, &full[s]);
          if (h) tma_3d(st + 2 * PB, &tmA3, r0, &full[s]);
        }
        for (int p = a.pwf; p < pw; ++p) {
          tma_2d(st + p * kG2Panel, &tmS, 32 * p, r0, &full[s]);
          if (h) tma_2d(st + 2 * PB + p * kG2Panel, &tmA, 32 * p, r0, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issue
    // A_hi x [B_hi | B_lo] (N = 64 pw: hi*hi and hi*lo side by side), then
    // A_lo x B_hi into the hi*lo columns: 2 MMAs per k-step, A_hi / B_hi read once
    const uint32_t idesc2 = idesc_tf32_mn(128, 64 * pw), idesc1 = idesc_tf32_mn(128, 32 * pw);
    const uint32_t base = smem_u32(sm);
    if (lane == 0)
      for (int t = 0; t < T; ++t) {
        const int s = t % kG2Stages, fg = t / kG2FL, buf = fg & 1;
        const bool first = (t % kG2FL) == 0, last = (t % kG2FL) == kG2FL - 1 || t == T - 1;
        if (first) mbar_wait(&tme[buf], ((fg >> 1) & 1) ^ 1);
        mbar_wait(&drv[s], (t / kG2Stages) & 1);
        tcf_after();
        const uint32_t st = base + (uint32_t)(s * SB);
        const uint32_t dHi = tbase + buf * 256, dX = dHi + 32 * pw;
#pragma unroll
        for (int ks = 0; ks < kG2TK / 8; ++ks) {
          const uint32_t o = ks * 1024;
          const uint64_t dAh = desc_sw128(st + o, kG2Panel, 512);
          const uint64_t dAl = desc_sw128(st + PB + o, kG2Panel, 512);
          const uint64_t dBh = desc_sw128(st + 2 * PB + o, kG2Panel, 512);  // [B_hi | B_lo]
          const uint32_t init = (first && ks == 0) ? 0u : 1u;
          if (!(a.dbg & 1)) {
            mma_tf32(dHi, dAh, dBh, idesc2, init);
            mma_tf32(dX, dAl, dBh, idesc1, 1u);
          }
        }
        mma_commit(&empty[s]);
        if (last) mma_commit(&tmf[buf]);
      }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- workers
    const int wt = tid - 64;                 // 0..255
    const int q = warp & 3;                  // TMEM lane quadrant (warp id % 4)
    const int ch = (warp - 2) >> 2;          // drained column half
    const int hw = 16 * pw;                  // columns per half
    const int nch = pw * kG2TK * 8;          // 16-byte chunks per pw-panel group
    const int i = 32 * q + lane;             // Gram row drained by this thread
    const int jmin = i & ~7;                 // block-upper part only
    double *dp = a.part + (narrow ? (size_t)pair : (size_t)pair * 2 + h) * 128 * 128;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.f;
    int drained = 0;
    for (int t = 0; t < T; ++t) {
      const int s = t % kG2Stages;
      mbar_wait(&full[s], (t / kG2Stages) & 1);
      unsigned char *st = sm + s * SB;
      for (int e = wt; e < ((a.dbg & 2) ? 0 : nch); e += 256) {
        const int o = e * 16;
        const float4 x = *reinterpret_cast<const float4 *>(st + o);
        float4 hi, lo;
        if (narrow) {
          // the upper panels of S also give the lower B panels (b S); the upper B panels are AS
          if (o >= (pw / 2) * kG2Panel) {
            const int ob = o - (pw / 2) * kG2Panel;
            const float br = sb[s * 32 + ((o % kG2Panel) >> 7)];
            split4(make_float4(br * x.x, br * x.y, br * x.z, br * x.w), hi, lo);
            *reinterpret_cast<float4 *>(st + 2 * PB + ob) = hi;
            *reinterpret_cast<float4 *>(st + 3 * PB + ob) = lo;
            split4(*reinterpret_cast<const float4 *>(st + 2 * PB + o), hi, lo);
            *reinterpret_cast<float4 *>(st + 2 * PB + o) = hi;
            *reinterpret_cast<float4 *>(st + 3 * PB + o) = lo;
          }
          split4(x, hi, lo);
          *reinterpret_cast<float4 *>(st + o) = hi;
          *reinterpret_cast<float4 *>(st + PB + o) = lo;
          continue;
        }
        if (h == 0) {
          const float br = sb[s * 32 + ((o % kG2Panel) >> 7)];  // 0 beyond n (TMA fill)
          split4(make_float4(br * x.x, br * x.y, br * x.z, br * x.w), hi, lo);
        } else {
          split4(*reinterpret_cast<const float4 *>(st + 2 * PB + o), hi, lo);
        }
        *reinterpret_cast<float4 *>(st + 2 * PB + o) = hi;  // B hi (bS, or AS in place)
        *reinterpret_cast<float4 *>(st + 3 * PB + o) = lo;  // B lo
        split4(x, hi, lo);
        *reinterpret_cast<float4 *>(st + o) = hi;           // S hi (in place)
        *reinterpret_cast<float4 *>(st + PB + o) = lo;      // S lo
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) arrive(&drv[s]);
      // drain group g two tiles after it closed (its MMAs have had time to finish)
      if (t % kG2FL == 1 && t > kG2FL)
        g2_drain(drained++, NG, tmf, tme, tbase, q, ch, hw, lane, i, narrow ? 0 : jmin, a.w, dp,
                 acc, a.dbg & 4, narrow, a.wneed);
    }
    while (drained < NG)
      g2_drain(drained++, NG, tmf, tme, tbase, q, ch, hw, lane, i, narrow ? 0 : jmin, a.w, dp, acc,
               a.dbg & 4, narrow, a.wneed);
  }
  tcf_before();
  __syncthreads();
  if (warp == 1) {
    tcf_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

// G (w x w row-major) from the CTA partials; block-lower 8x8 blocks mirrored
__global__ void k_reduce_gram_tc2(const double *__restrict__ part, int nct, int w,
                                  double *__restrict__ GB, double *__restrict__ GA) {
  const int tot = 2 * w * w;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int g = e / (w * w);
    const int r = e - g * w * w;
    int i = r / w, j = r - i * w;
    if ((i >> 3) > (j >> 3)) {
      const int t = i;
      i = j;
      j = t;
    }
    double s = 0.0;
    for (int c = 0; c < nct; ++c) s += part[(((size_t)c * 2 + g) * 128 + j) * 128 + i];
    (g ? GA : GB)[r] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    MG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    require(p != nullptr && q == cudaDriverEntryPointSuccess, MG_ERR_CUDA,
            "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// row-major fp32 [n x ld], columns [0, w): 32-column x kG2TK-row SW128 boxes
CUtensorMap make_map(const float *base, int64_t n, int ld, int w) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {32, (cuuint32_t)kG2TK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MG_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// the first pf full 32-column panels of row-major fp32 [n x ld] as a 3-D
// tensor (column-in-panel, row, panel): one box = kG2TK rows x pf panels,
// landing panel-major exactly like pf separate 2-D boxes
CUtensorMap make_map_3d(const float *base, int64_t n, int ld, int pf) {
  CUtensorMap m;
  const int pd = pf > 0 ? pf : 1;
  cuuint64_t dims[3] = {32, (cuuint64_t)n, (cuuint64_t)pd};
  cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(float), 32 * sizeof(float)};
  cuuint32_t box[3] = {32, (cuuint32_t)kG2TK, (cuuint32_t)pd};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MG_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return m;
}

// fp32 vector [n]: kG2TK-element boxes (zero beyond n)
CUtensorMap make_map_1d(const float *base, int64_t n) {
  CUtensorMap m;
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t strides[1] = {0};
  cuuint32_t box[1] = {(cuuint32_t)kG2TK};
  cuuint32_t es[1] = {1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<float *>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MG_ERR_CUDA, "cuTensorMapEncodeTiled (1-D) failed: " + std::to_string((int)r));
  return m;
}

}  // namespace

// W-column blocks from the narrow kernel's partials (hb = 32 pw / 2 columns per
// half): B column j < hb is G_B[i][hb + j], j >= hb is G_A[i][j]; rows i < w,
// W columns [2mp, w).
// Written with the full kernel's mirror convention (block-lower 8 x 8 blocks
// come from the block-upper product), and mirrored into the W rows.
__global__ void k_reduce_gram_w(const double *__restrict__ part, int nct, int w, int mp, int hb,
                                double *__restrict__ GB, double *__restrict__ GA) {
  const int nw = w - 2 * mp;
  const int tot = 2 * w * nw;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int g = e / (w * nw);
    const int r = e - g * w * nw;
    int i = r / nw, j = 2 * mp + (r - i * nw);  // target entry (i, j), j a W column
    const int ti = i, tj = j;
    if ((i >> 3) > (j >> 3)) {  // block-lower inside the W x W block: take the mirror product
      const int t = i;
      i = j;
      j = t;
    }
    double s = 0.0;
    for (int c = 0; c < nct; ++c) s += part[((size_t)c * 128 + (g * hb + j - hb)) * 128 + i];
    double *G = g ? GA : GB;
    G[ti * w + tj] = s;
    if (ti < 2 * mp) G[tj * w + ti] = s;  // W rows x [X P] columns
  }
}

bool gram_tc2_supported(int w, int ld) {
  return w > 32 && w <= 128 && ld % 4 == 0 && w % 4 == 0;
}

void gram_pair_tc2(mg_ctx *ctx, int64_t n, int ld, int w, const float *S, const float *AS,
                   const float *b, double *GB, double *GA, DBuf<double> &part) {
  require(gram_tc2_supported(w, ld), MG_ERR_INTERNAL, "tc2 Gram: unsupported width");
  require(((uintptr_t)S % 16) == 0 && ((uintptr_t)AS % 16) == 0, MG_ERR_INTERNAL,
          "tc2 Gram: operands must be 16-byte aligned");
  const int pw = (w + 31) / 32;
  const int64_t ntiles = (n + kG2TK - 1) / kG2TK;
  const int npairs = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms / 2));
  const int grid = 2 * npairs;
  const size_t need = (size_t)grid * 128 * 128;
  if (part.n < need) part.alloc(ctx, need);
  MG_CUDA(cudaMemsetAsync(part.p, 0, need * sizeof(double), ctx->stream));
  Gram2TcArgs a{};
  a.n = n;
  a.w = w;
  a.pw = pw;
  a.npairs = npairs;
  a.part = part.p;
  {
    const char *e = getenv("MG_TC2_DBG");
    a.dbg = e ? atoi(e) : 0;
  }
  a.pwf = w / 32;
  const CUtensorMap mS = make_map(S, n, ld, w), mA = make_map(AS, n, ld, w), mB = make_map_1d(b, n);
  const CUtensorMap mS3 = make_map_3d(S, n, ld, a.pwf), mA3 = make_map_3d(AS, n, ld, a.pwf);
  const size_t smem = g2_smem_bytes(pw);
  static thread_local size_t smem_set = 0;
  if (smem > smem_set) {
    MG_CUDA(cudaFuncSetAttribute(k_gram_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    smem_set = smem;
  }
  {
    ProfScope ps(ctx, PROF_GRAM, 2.0 * n * w * sizeof(float) + 4.0 * n);
    k_gram_tc2<<<grid, kG2Threads, smem, ctx->stream>>>(mS, mA, mS3, mA3, mB, a);
    MG_CHECK_LAUNCH(ctx);
  }
  k_reduce_gram_tc2<<<grid_for(2 * w * w, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
      part.p, npairs, w, GB, GA);
  MG_CHECK_LAUNCH(ctx);
}

// W-column blocks only: G_B[:, W] = S' (b W), G_A[:, W] = S' (A W) and their
// mirrors (rows W x columns [X P]); the [X P] x [X P] blocks are left untouched
// (the caller derives them from the previous step's Grams).  w = 108 (mp = 36) or w = 60 (mp = 20).
bool gram_w_tc2_supported(int w, int mp, int ld) {
  const int pw = (w + 31) / 32;
  return gram_tc2_supported(w, ld) && pw % 2 == 0 && 2 * mp >= 32 * (pw / 2) && w == 3 * mp;
}

void gram_w_tc2(mg_ctx *ctx, int64_t n, int ld, int w, int mp, const float *S, const float *AS,
                const float *b, double *GB, double *GA, DBuf<double> &part) {
  require(gram_w_tc2_supported(w, mp, ld), MG_ERR_INTERNAL, "narrow tc2 Gram: unsupported width");
  const int pw = (w + 31) / 32, hb = 32 * (pw / 2);
  const int64_t ntiles = (n + kG2TK - 1) / kG2TK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms));
  const size_t need = (size_t)grid * 128 * 128;
  if (part.n < need) part.alloc(ctx, need);
  MG_CUDA(cudaMemsetAsync(part.p, 0, need * sizeof(double), ctx->stream));
  Gram2TcArgs a{};
  a.n = n;
  a.w = w;
  a.pw = pw;
  a.npairs = grid;
  a.part = part.p;
  a.narrow = 1;
  a.wneed = (w - hb + 15) / 16 * 16;
  a.pwf = w / 32;
  const CUtensorMap mS = make_map(S, n, ld, w), mA = make_map(AS, n, ld, w), mB = make_map_1d(b, n);
  const CUtensorMap mS3 = make_map_3d(S, n, ld, a.pwf), mA3 = make_map_3d(AS, n, ld, a.pwf);
  const size_t smem = g2_smem_bytes(pw);
  static thread_local size_t smem_set = 0;
  if (smem > smem_set) {
    MG_CUDA(cudaFuncSetAttribute(k_gram_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    smem_set = smem;
  }
  {
    ProfScope ps(ctx, PROF_GRAM, (double)n * (w + (w - 2 * mp)) * sizeof(float) + 4.0 * n);
    k_gram_tc2<<<grid, kG2Threads, smem, ctx->stream>>>(mS, mA, mS3, mA3, mB, a);
    MG_CHECK_LAUNCH(ctx);
  }
  k_reduce_gram_w<<<grid_for(2 * w * (w - 2 * mp), 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
      part.p, grid, w, mp, hb, GB, GA);
  MG_CHECK_LAUNCH(ctx);
}

}  // namespace mg
