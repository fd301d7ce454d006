// tcgen05 LOBPCG update (fp32 solve, wide blocks): the reference's
//   P = S Zp,  X = X Yx + P   (and the same for the A-images, eigensolver.py:255-258)
// followed by the fused residual R = AX - B X Theta, W = D^-1 R and the column
// norms, as ONE tensor-core pass over S = [X | P | W] and AS.
//
// Numerics (profiles/r2_update_tc.md).  Round 1 put X Yx itself on the tensor
// core and paid +15 % .. +210 % LOBPCG iterations: every product of the
// dominant term X_c Yx_cc ~ X_c was rounded to 2^-22 and accumulated without
// round-to-nearest.  Here the tensor core only forms the CORRECTION
//   dX = S (Zp + [Yx - I; 0; 0]),   dAX = AS (same),   P = S Zp,   AP = AS Zp
// and the epilogue adds it to the old X / AX in fp32 (X_new = X_old + dX, one
// rounding).  Near convergence |dX| << |X|, so the 2-piece TF32 products
// (2^-22 relative to dX) and the tensor core's accumulation are far below one
// fp32 ulp of X.  Emulated first (MG_UPD_EMUL in k_update_resid): iteration
// counts within the run-to-run spread of the fp32 FMA update.
//
// Shape.  The product is formed TRANSPOSED: D[j][r] = sum_k Z2[k][j] S[r][k],
//   A operand = Z2' (M = 2mp output columns, padded by the hardware to 128 lanes;
//               K-major SWIZZLE_128B, built once per CTA, hi / lo pieces),
//   B operand = a 128-row tile of S or AS (N = 128 rows, K = 32 columns per
//               box), in the layout TMA lands it (SWIZZLE_128B boxes): two
//               splitter warps round it in place, hi = rn_tf32(x), and write
//               lo = rn_tf32(x - hi) (with the hardware's truncation as hi the
//               dropped lo*lo term is a one-signed 2^-22: P = S Zp cancels
//               ~50x, and the solve diverged at iteration ~270 of C5-2M).
// So TMEM lane j holds output column j for the 128 rows of the tile: an
// epilogue warp's stores are 128-byte coalesced rows of X / P / W / AX / AP,
// and the column sums (residual and X norms) are per-thread fp64 chains.
// The coefficients are rounded to TF32 ONCE (Z2' -> rn_tf32): the same rounded
// matrix multiplies S and AS, so X and its A-image stay consistent and the
// step is merely 2^-12-inexact in the (small) corrections -- an inexact line
// search, which LOBPCG tolerates and the next Rayleigh-Ritz absorbs.  That
// leaves 2 MMAs per k-step (Z2' x lo, Z2' x hi) instead of 3.  Z2' lives in
// TMEM (A operand, 112 columns); the accumulators are double-buffered there
// (2 x [D_S 96 | D_AS 96] columns).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "mg_fastk.cuh"
#include "mg_tc.cuh"

namespace mg {

namespace {

constexpr int kU3Threads = 512;
constexpr int kU3Rows = 96;            // rows per tile (MMA N)
constexpr int kU3Box = kU3Rows * 128;  // bytes of one 32-column box
constexpr int kU3NR = 2;               // raw matrix-tile ring
constexpr int kU3NL = 4;               // lo box ring
constexpr int kU3Acc = 128;            // TMEM column of the accumulators (Z2' sits below)

__host__ __device__ constexpr size_t u3_xbytes(int mp) {
  return ((size_t)2 * kU3Rows * mp * 4 + 127) / 128 * 128;  // old X and AX columns of a tile
}
// output staging per row group: 16 complete rows of [X P W] (3mp), [AX AP]
// (2mp) and compact W (mp)
__host__ __device__ constexpr size_t u3_obytes(int mp) { return (size_t)16 * 6 * mp * 4; }
__host__ __device__ constexpr size_t u3_smem(int np, int mp) {
  return (size_t)kU3NR * np * kU3Box + (size_t)kU3NL * kU3Box + u3_xbytes(mp) +
         3 * u3_obytes(mp) + 512;
}

// K-major SWIZZLE_128B operand (8-row x 128-byte atoms, SBO = 1024)
__device__ __forceinline__ uint64_t desc_k128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// D f32, A/B tf32, both K-major
__host__ __device__ constexpr uint32_t idesc_tf32_k(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] B[smem]
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
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
__device__ __forceinline__ void tma_st2d(const CUtensorMap *map, int c0, int r0, const void *src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(r0), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t ta, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t ta, const float *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(ta),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
// round to nearest (ties away) TF32 of a finite value (cvt.rna.tf32.f32 expands
// to a multi-instruction sequence on sm_100; the integer form is two)
__device__ __forceinline__ float rn_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

struct Upd3Args {
  int64_t n;
  int m;
  const int *skip;   // device flag: nonzero -> return (fallback iteration)
  double *part;      // [grid][2*mp] column partials (sum r^2, sum x^2)
  float *wc;         // compact W, the SpMM input: n x wcs, columns = physical W columns
                     // [wc0, wc0 + wcs) (wcs = mp, wc0 = 0: the whole block)
  int wcs, wc0;
  int perm[40];      // physical W column of logical column c (identity unless the solver
                     // packs the unconverged columns into a suffix)
  int dbg;           // MG_U3_DBG timing experiments: 1 no MMA, 2 no split, 4 no epilogue I/O
};

// the solver's row stride for a block of mp columns (Lobpcg::Lobpcg, mg_lobpcg.cu)
__host__ __device__ constexpr int u3_ld(int mp) {
  return ((3 * mp + 4) / 4) % 2 == 0 ? 3 * mp + 8 : 3 * mp + 4;
}

// spin with a short sleep: the waiting producer / issuer lanes share their
// scheduler with epilogue warps
__device__ int g_u3_nosleep = 0;
__device__ __forceinline__ void mbar_wait_bk(uint64_t *bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.b32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(phase)
        : "memory");
    if (ok) break;
    if (!g_u3_nosleep) __nanosleep(32);
  }
}

// Warp roles (16 warps; warp w runs on scheduler w % 4, and only warps with
// w % 4 == q can read TMEM lanes 32q .. 32q + 31):
//   epilogue  0, 4, 8 (q = 0)   1, 5, 9 (q = 1)   2, 6, 10 (q = 2)   [lane = output column;
//             three row groups of 32 rows: the per-chunk dependency chain, not the
//             instruction count, bounds a warp, so more warps in flight pay]
//   splitters 13, 14, 7, 11   TMA producers 3 (tiles), 12 (old X / AX)   MMA issuer 15
template <int MP>
__global__ void __launch_bounds__(kU3Threads, 1)
    k_update_tc3(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmA,
                 const __grid_constant__ CUtensorMap tmXS, const __grid_constant__ CUtensorMap tmXA,
                 const __grid_constant__ CUtensorMap tmOS, const __grid_constant__ CUtensorMap tmOA,
                 const __grid_constant__ CUtensorMap tmOW, float *S, float *AS, const float *__restrict__ b,
                 const float *__restrict__ prec, const float *__restrict__ Mg,
                 const double *__restrict__ theta, Upd3Args a) {
  if (*a.skip) return;
  constexpr int LD = u3_ld(MP), W = 3 * MP, NP = (W + 31) / 32, KS = (W + 7) / 8;
  constexpr int NQ = (2 * MP + 31) / 32;          // TMEM lane quadrants holding output columns
  constexpr uint32_t MT = (uint32_t)NP * kU3Box;  // bytes of one matrix tile (NP boxes)
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char *raw = sm;
  unsigned char *los = raw + (size_t)kU3NR * MT;
  float *xbuf = reinterpret_cast<float *>(los + (size_t)kU3NL * kU3Box);  // [2][rows][MP]
  float *obuf = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(xbuf) +
                                          u3_xbytes(MP));  // [row group]
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(obuf) +
                                                3 * u3_obytes(MP));
  uint64_t *full = bars, *rempty = full + kU3NR, *lfull = rempty + kU3NR, *lempty = lfull + kU3NL;
  constexpr int NG = 3;                   // epilogue row groups (32 rows of a tile each)
  constexpr int NC = kU3Rows / (16 * NG);  // 16-row chunks per tile and row group
  constexpr int NX = NG * NC;              // X staging slots: one per (row group, chunk)
  uint64_t *afull = lempty + kU3NL, *aempty = afull + 2, *xfull = aempty + 2, *xempty = xfull + NX;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(xempty + NX);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (a.n + kU3Rows - 1) / kU3Rows;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int T = (int)(t_end - t_begin);

  // compact-W slots beyond the block's last column are never written: keep them zero
  for (int e = tid; e < (int)(3 * u3_obytes(MP) / 4); e += kU3Threads) obuf[e] = 0.f;
  if (tid == 0) {
    for (int s = 0; s < kU3NR; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&rempty[s], 1);
    }
    for (int s = 0; s < kU3NL; ++s) {
      mbar_init(&lfull[s], 4);
      mbar_init(&lempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], NG * NQ);
    }
    for (int s = 0; s < NX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], NQ);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 15) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tcf_before();
  __syncthreads();
  tcf_after();
  const uint32_t tbase = *tslot;
  if ((smem_u32(sm) & 1023) != 0) __trap();

  // A operand in TMEM (lane j = output column, TMEM column k): Z2'(j, k),
  //   j < mp:        Zp[k][j] + (k < mp ? Yx[k][j] - delta_kj : 0)   (correction of X column j)
  //   mp <= j < 2mp: Zp[k][j - mp]                                    (P column)
  // as hi = rn_tf32 and lo = rn_tf32(v - hi) pieces; other lanes are zero.
  if (warp >= 4 && warp < 8) {
    const int j = 32 * (warp & 3) + lane;
    const int c = j < MP ? j : j - MP;
    const uint32_t tz = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int k0 = 0; k0 < 8 * KS; k0 += 16) {
      float hi[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int k = k0 + e;
        float v = 0.f;
        if (k < W && j < 2 * MP) {
          v = Mg[k * MP + c];
          if (j < MP && k < MP) v += Mg[W * MP + k * MP + c] - (k == c ? 1.f : 0.f);
        }
        hi[e] = rn_tf32(v);
      }
      tmem_st16(tz + k0, hi);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tcf_before();
  __syncthreads();
  tcf_after();

  const int q = warp & 3;
  if (warp == 3) {
    // --------------------------------------------------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmS)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      uint32_t g = 0;
      for (int ti = 0; ti < T; ++ti) {
        const int r0 = (int)((t_begin + ti) * kU3Rows);
        for (int mat = 0; mat < 2; ++mat, ++g) {
          const int s = g % kU3NR;
          mbar_wait_bk(&rempty[s], ((g / kU3NR) & 1) ^ 1);
          mbar_expect_tx(&full[s], MT);
#pragma unroll
          for (int p = 0; p < NP; ++p)
            tma_2d(raw + (size_t)s * MT + (size_t)p * kU3Box, mat ? &tmA : &tmS, 32 * p, r0,
                   &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 15) {
    // ------------------------------------------------------------ MMA issue
    constexpr uint32_t idesc = idesc_tf32_k(128, kU3Rows);
    const uint32_t rb = smem_u32(raw), lb = smem_u32(los);
    if (lane == 0) {
      uint32_t g = 0;
      for (int ti = 0; ti < T; ++ti) {
        const int buf = ti & 1;
        mbar_wait_bk(&aempty[buf], ((ti >> 1) & 1) ^ 1);
        tcf_after();
        for (int mat = 0; mat < 2; ++mat, ++g) {
          const int s = g % kU3NR;
          const uint32_t d = tbase + kU3Acc + buf * (2 * kU3Rows) + mat * kU3Rows;
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const uint32_t gb = g * NP + p;
            const int j = gb % kU3NL;
            mbar_wait_bk(&lfull[j], (gb / kU3NL) & 1);  // hi (in place) and lo of this box
            tcf_after();
            if (!(a.dbg & 1)) {
#pragma unroll
              for (int ks = 4 * p; ks < 4 * p + 4 && ks < KS; ++ks) {
                const uint32_t off = (ks & 3) * 32;
                const uint64_t dBh = desc_k128(rb + s * MT + p * kU3Box + off);
                const uint64_t dBl = desc_k128(lb + j * kU3Box + off);
                const uint32_t aH = tbase + 8 * ks;
                // small products first
                mma_tf32_ts(d, aH, dBl, idesc, ks == 0 ? 0u : 1u);
                mma_tf32_ts(d, aH, dBh, idesc, 1u);
              }
            }
            mma_commit(&lempty[j]);
          }
          mma_commit(&rempty[s]);
        }
        mma_commit(&afull[buf]);
      }
    }
    __syncwarp();
  } else if (warp == 12) {
    // ---------------------------------- old X / AX columns for the epilogue
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmXS)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmXA)) : "memory");
      // one slot per (row half, 16-row chunk): a slot is refilled for the next
      // tile as soon as its NQ reader warps have taken their values
      for (int ti = 0; ti < T; ++ti)
        for (int ch = 0; ch < NC; ++ch)
          for (int hf = 0; hf < NG; ++hf) {
            const int sl = hf * NC + ch;
            const int r0 = (int)((t_begin + ti) * kU3Rows) + hf * (kU3Rows / NG) + ch * 16;
            float *dst = xbuf + sl * (2 * 16 * MP);
            mbar_wait_bk(&xempty[sl], (ti & 1) ^ 1);
            mbar_expect_tx(&xfull[sl], 2 * 16 * MP * 4);
            tma_2d(dst, &tmXS, 0, r0, &xfull[sl]);
            tma_2d(dst + 16 * MP, &tmXA, 0, r0, &xfull[sl]);
          }
    }
    __syncwarp();
  } else if (warp == 13 || warp == 14 || warp == 7 || warp == 11) {
    // ------------------------------------------------------------ splitters
    // hi = rn_tf32(x) in place, lo = rn_tf32(x - hi); 16-byte chunks whose
    // columns lie beyond the last k-step are skipped (128-byte rows, chunk
    // XOR-swizzled with the row)
    const int st = (warp == 13 ? 0 : warp == 14 ? 1 : warp == 7 ? 2 : 3) * 32 + lane;  // 0..127
    constexpr int nchunk = kU3Box / 16;  // per box: 6 per thread
    uint32_t g = 0;
    for (int ti = 0; ti < T; ++ti)
      for (int mat = 0; mat < 2; ++mat, ++g) {
        const int s = g % kU3NR;
        mbar_wait_bk(&full[s], (g / kU3NR) & 1);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const uint32_t gb = g * NP + p;
          const int j = gb % kU3NL;
          mbar_wait_bk(&lempty[j], ((gb / kU3NL) & 1) ^ 1);
          float4 *src = reinterpret_cast<float4 *>(raw + (size_t)s * MT + (size_t)p * kU3Box);
          float4 *dst = reinterpret_cast<float4 *>(los + (size_t)j * kU3Box);
          if (!(a.dbg & 2)) {
            float4 x[nchunk / 128];
#pragma unroll
            for (int i = 0; i < nchunk / 128; ++i) x[i] = src[st + 128 * i];
#pragma unroll
            for (int i = 0; i < nchunk / 128; ++i) {
              const int e = st + 128 * i, ck = (e & 7) ^ ((e >> 3) & 7);
              if (32 * p + 4 * ck >= 8 * KS) continue;
              const float4 h = make_float4(rn_tf32(x[i].x), rn_tf32(x[i].y), rn_tf32(x[i].z),
                                           rn_tf32(x[i].w));
              src[e] = h;
              // lo = x - hi is exact in fp32; the tensor core reads its top 11 bits
              // (|lo| <= 2^-12 |x|: what it drops is below 2^-23 |x|, of either sign)
              dst[e] = make_float4(x[i].x - h.x, x[i].y - h.y, x[i].z - h.z, x[i].w - h.w);
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) arrive(&lfull[j]);
        }
      }
  } else if (warp < 12 && q < NQ) {
    // ------------------------------------------------------------- epilogue
    // Chunks of 16 rows, software-pipelined: the old X / AX values and b / prec
    // of chunk u + 1 are loaded before chunk u is drained, so one L2 round
    // trip is hidden behind a chunk of arithmetic and stores.  LD is a
    // compile-time constant: every row address is base + immediate.
    const int half = warp >> 2;  // row group
    const int j = 32 * q + lane;           // output column held by this TMEM lane
    const bool isx = j < MP;
    const int c = isx ? j : j - MP;
    const bool live = j < 2 * MP && c < a.m;   // pad columns stay zero: never written
    const bool actx = isx && live, actp = !isx && live;
    const float th = actx ? (float)theta[c] : 0.f;
    double sr = 0.0, sx = 0.0;
    const int64_t NU = (int64_t)T * NC;
    auto row_of = [&](int64_t u) {
      return (t_begin + u / NC) * kU3Rows + half * (kU3Rows / NG) + (int)(u % NC) * 16;
    };
    float bn = 0.f, pn = 1.f;  // next chunk's b / prec (lane & 15 holds row rr + (lane & 15))
    auto load_bp = [&](int64_t u) {
      const int64_t rl = row_of(u) + (lane & 15);
      bn = rl < a.n ? __ldg(b + rl) : 0.f;
      pn = (prec && rl < a.n) ? __ldg(prec + rl) : 1.f;
    };
    const bool on = !(a.dbg & 4);
    if (on && NU > 0) load_bp(0);
    for (int64_t u = 0; u < NU; ++u) {
      const int ti = (int)(u / NC), ch = (int)(u % NC), buf = ti & 1;
      const float bc = bn, pc = pn;
      if (on && u + 1 < NU) load_bp(u + 1);
      float xo[16], ao[16];
      {
        // old X / AX columns of this chunk, staged by TMA (exact fp32)
        const int sl = half * NC + ch;
        if (!(a.dbg & 64)) mbar_wait_bk(&xfull[sl], ti & 1);
        const float *xs = xbuf + sl * (2 * 16 * MP) + c;
        if (actx) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            xo[e] = xs[e * MP];
            ao[e] = xs[16 * MP + e * MP];
          }
        }
        __syncwarp();
        if (lane == 0) arrive(&xempty[sl]);  // refilled for the next tile meanwhile
      }
      if (ch == 0) {
        mbar_wait_bk(&afull[buf], (ti >> 1) & 1);
        __syncwarp();
        tcf_after();
      }
      if (on) {
        const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + kU3Acc + buf * (2 * kU3Rows) +
                            half * (kU3Rows / NG) + ch * 16;
        float dS[16], dA[16];
        if (!(a.dbg & 16)) {
          tmem_ld16(ta, dS);
          tmem_ld16(ta + kU3Rows, dA);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) dS[e] = dA[e] = 0.f;
        }
        // Outputs are staged as complete rows in shared memory (lane = column:
        // conflict-free) and written by TMA: row-contiguous 432 / 288 / 144-byte
        // segments, ~10 L2 line transactions per row.  Per-warp 128-byte stores
        // of single column blocks cost ~18 and bounded the kernel (3.6 ms of
        // 9.4 at C5).  Rows beyond n are clipped by the tensor maps.
        float *oS = obuf + (size_t)half * (16 * 6 * MP);
        float *oA = oS + 16 * W, *oW = oA + 16 * 2 * MP;
        const int wcs = a.wcs;
        if (q == 0 && lane == 0)  // the previous chunk's stores have read the slot
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync %0, %1;" ::"r"(2 + half), "n"(32 * NQ) : "memory");
        // b / prec are uniform per row: shuffled before the lanes split into roles
        float br[16], pr[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          br[e] = __shfl_sync(0xffffffffu, bc, e) * th;
          pr[e] = __shfl_sync(0xffffffffu, pc, e);
        }
        const int64_t rr = row_of(u);
        const int nrow = (a.dbg & 8) ? 0 : (int)max((int64_t)0, min((int64_t)16, a.n - rr));
        if (isx) {
          const int pc = a.perm[c];  // W's physical column, and its slot in the compact block
          const int pcw = (pc >= a.wc0 && pc - a.wc0 < wcs) ? pc - a.wc0 : -1;
          float s1 = 0.f, s2 = 0.f;  // fp32 over the chunk's 16 rows, fp64 across chunks
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x1 = 0.f, a1 = 0.f, wv = 0.f;  // pad columns stay zero
            if (actx) {
              x1 = xo[e] + dS[e];
              a1 = ao[e] + dA[e];
              const float r = a1 - br[e] * x1;
              if (e < nrow) {
                s1 = fmaf(r, r, s1);
                s2 = fmaf(x1, x1, s2);
              }
              wv = pr[e] * r;
            }
            oS[e * W + c] = x1;
            oA[e * 2 * MP + c] = a1;
            oS[e * W + 2 * MP + pc] = wv;
            if (pcw >= 0) oW[e * wcs + pcw] = wv;
          }
          sr += (double)s1;
          sx += (double)s2;
        } else if (j < 2 * MP) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            oS[e * W + MP + c] = actp ? dS[e] : 0.f;
            oA[e * 2 * MP + MP + c] = actp ? dA[e] : 0.f;
          }
        }
        fence_proxy_async();
        asm volatile("bar.sync %0, %1;" ::"r"(2 + half), "n"(32 * NQ) : "memory");
        if (q == 0 && lane == 0) {
          if (nrow > 0) {
            tma_st2d(&tmOS, 0, (int)rr, oS);
            tma_st2d(&tmOA, 0, (int)rr, oA);
            tma_st2d(&tmOW, 0, (int)rr, oW);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (ch == NC - 1) {
        tcf_before();
        __syncwarp();
        if (lane == 0) arrive(&aempty[buf]);
      }
    }
    if (q == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    // column partials: the row groups of a column meet in shared memory
    // (the raw ring is idle by now: every box was consumed before the last afull)
    double *red = reinterpret_cast<double *>(raw);
    if (isx) {
      red[(half * MP + c) * 2] = sr;
      red[(half * MP + c) * 2 + 1] = sx;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * NG * NQ) : "memory");
    if (half == 0 && isx) {
      double t1 = 0.0, t2 = 0.0;
      for (int g2 = 0; g2 < NG; ++g2) {
        t1 += red[(g2 * MP + c) * 2];
        t2 += red[(g2 * MP + c) * 2 + 1];
      }
      a.part[(size_t)blockIdx.x * 2 * MP + c] = t1;
      a.part[(size_t)blockIdx.x * 2 * MP + MP + c] = t2;
    }
  }
  tcf_before();
  __syncthreads();
  if (warp == 15) {
    tcf_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn3() {
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

// row-major fp32 [n x ld], columns [0, w): 32-column x 128-row SWIZZLE_128B
// boxes = the K-major tf32 operand atoms (columns >= w and rows >= n read 0)
CUtensorMap make_map_k(const float *base, int64_t n, int ld, int w) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {32, (cuuint32_t)kU3Rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn3()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MG_ERR_CUDA,
          "cuTensorMapEncodeTiled (update) failed: " + std::to_string((int)r));
  return m;
}

// columns [0, cols) of row-major fp32 [n x ld]: bw-column x 16-row boxes,
// unswizzled (the epilogue's exact old X / AX values, and its output blocks)
CUtensorMap make_map_x(const float *base, int64_t n, int ld, int cols, int bw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)bw, 16};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn3()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MG_ERR_CUDA,
          "cuTensorMapEncodeTiled (update, X block) failed: " + std::to_string((int)r));
  return m;
}

}  // namespace

bool update_tc3_supported(int w, int mp, int ld) {
  return (mp == 12 || mp == 20 || mp == 36) && w == 3 * mp && ld == u3_ld(mp);
}

template <int MP>
static void launch_tc3(mg_ctx *ctx, int grid, const CUtensorMap &mS, const CUtensorMap &mA,
                       const CUtensorMap &mXS, const CUtensorMap &mXA, const CUtensorMap &mOS,
                       const CUtensorMap &mOA, const CUtensorMap &mOW, float *S, float *AS, const float *b, const float *prec, const float *Mg,
                       const double *theta, const Upd3Args &a) {
  constexpr size_t smem = u3_smem((3 * MP + 31) / 32, MP);
  static_assert(smem <= 227 * 1024, "tc update: shared memory");
  static thread_local bool attr_set = false;
  if (!attr_set) {
    MG_CUDA(cudaFuncSetAttribute(k_update_tc3<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_set = true;
  }
  k_update_tc3<MP><<<grid, kU3Threads, smem, ctx->stream>>>(mS, mA, mXS, mXA, mOS, mOA, mOW, S, AS,
                                                            b, prec, Mg, theta, a);
}

// one fast-path update on the tensor cores; part: [grid][2 mp]; returns the grid
int update_tc3(mg_ctx *ctx, int64_t n, int ld, int w, int m, int mp, float *S, float *AS,
               const float *b, const float *prec, const float *Mg, const double *theta,
               const int *skip, double *part, float *wc, const int *perm, int wc0, int wcs) {
  require(update_tc3_supported(w, mp, ld), MG_ERR_INTERNAL, "tc update: unsupported shape");
  require(((uintptr_t)S % 16) == 0 && ((uintptr_t)AS % 16) == 0, MG_ERR_INTERNAL,
          "tc update: operands must be 16-byte aligned");
  Upd3Args a{};
  a.n = n;
  a.m = m;
  a.skip = skip;
  a.part = part;
  a.wc = wc;
  require(wcs >= 4 && wcs <= mp && wcs % 4 == 0 && wc0 >= 0 && wc0 + wcs <= mp + 32, MG_ERR_INTERNAL,
          "tc update: bad compact W layout");
  a.wcs = wcs;
  a.wc0 = wc0;
  for (int c = 0; c < 40; ++c) a.perm[c] = (perm && c < mp) ? perm[c] : c;
  {
    const char *e = getenv("MG_U3_DBG");
    a.dbg = e ? atoi(e) : 0;
    const int ns = (a.dbg & 32) ? 1 : 0;
    MG_CUDA(cudaMemcpyToSymbolAsync(g_u3_nosleep, &ns, sizeof(int), 0, cudaMemcpyHostToDevice,
                                    ctx->stream));
  }
  const int64_t ntiles = (n + kU3Rows - 1) / kU3Rows;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms));
  const CUtensorMap mS = make_map_k(S, n, ld, w), mA = make_map_k(AS, n, ld, w);
  const CUtensorMap mXS = make_map_x(S, n, ld, mp, mp), mXA = make_map_x(AS, n, ld, mp, mp);
  // outputs: [X P W] of S, [AX AP] of AS, compact W (16-row boxes of complete rows)
  const CUtensorMap mOS = make_map_x(S, n, ld, 3 * mp, 3 * mp);
  const CUtensorMap mOA = make_map_x(AS, n, ld, 2 * mp, 2 * mp);
  const CUtensorMap mOW = make_map_x(wc, n, wcs, wcs, wcs);
  if (mp == 12)
    launch_tc3<12>(ctx, grid, mS, mA, mXS, mXA, mOS, mOA, mOW, S, AS, b, prec, Mg, theta, a);
  else if (mp == 20)
    launch_tc3<20>(ctx, grid, mS, mA, mXS, mXA, mOS, mOA, mOW, S, AS, b, prec, Mg, theta, a);
  else
    launch_tc3<36>(ctx, grid, mS, mA, mXS, mXA, mOS, mOA, mOW, S, AS, b, prec, Mg, theta, a);
  MG_CHECK_LAUNCH(ctx);
  return grid;
}

// One fast-path update through either kernel (C ABI mg_update_f32: unit tests
// and tools/bench_update.py).  variant 0: k_update_ws (fp32 FMA), 1: tcgen05.
// colsums (device, 2 mp): sum r^2 then sum x^2 per column.
namespace {
__global__ void k_sum_parts(const double *__restrict__ part, int nb, int w, double *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= w) return;
  double s = 0.0;
  for (int q = 0; q < nb; ++q) s += part[(size_t)q * w + t];
  out[t] = s;
}
}  // namespace

void update_f32_hook(mg_ctx *ctx, int variant, int64_t n, int ld, int m, int mp, float *S,
                     float *AS, const float *b, const float *prec, const float *Mg,
                     const double *theta, float *wc, double *colsums) {
  const int w = 3 * mp;
  DBuf<int> skip(ctx, 1);
  skip.zero();
  DBuf<double> part(ctx, (size_t)ctx->num_sms * 2 * mp);
  int nb;
  if (variant == 1) {
    nb = update_tc3(ctx, n, ld, w, m, mp, S, AS, b, prec, Mg, theta, skip.p, part.p, wc, nullptr, 0,
                    mp);
  } else {
    int tk = 0;
    for (int t = 256; t >= 32; t -= 4)
      if (upd_ws_bytes(t, ld, w, mp) <= 225 * 1024) {
        tk = t;
        break;
      }
    require(tk > 0 && mp % 4 == 0, MG_ERR_INPUT, "update hook: block too wide for k_update_ws");
    const size_t smem = upd_ws_bytes(tk, ld, w, mp);
    MG_CUDA(cudaFuncSetAttribute(k_update_ws<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    UpdArgs ua{};
    ua.n = n;
    ua.tk = tk;
    ua.ld = ld;
    ua.w = w;
    ua.m = m;
    ua.mp = mp;
    ua.skip = skip.p;
    ua.part = part.p;
    ua.wc = wc;
    nb = (int)std::min<int64_t>((n + tk - 1) / tk, ctx->num_sms);
    k_update_ws<4><<<nb, kWsF + kWsS, smem, ctx->stream>>>(S, AS, b, prec, Mg, theta, ua);
    MG_CHECK_LAUNCH(ctx);
  }
  k_sum_parts<<<(2 * mp + 63) / 64, 64, 0, ctx->stream>>>(part.p, nb, 2 * mp, colsums);
  MG_CHECK_LAUNCH(ctx);
}

}  // namespace mg
