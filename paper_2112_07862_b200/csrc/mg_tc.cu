// tcgen05 Gram pair: kernels and host side (design notes in mg_tc.cuh).
#include "mg_fastk.cuh"
#include "mg_tc.cuh"

namespace mg {

static constexpr int kTcThreads = 320;  // 10 warps: producer, MMA, 8 workers
static constexpr int kTcM = 128;        // Gram rows (S columns), zero-padded
static constexpr int kTcN = 64;         // Gram columns per CTA (half), zero-padded
static constexpr int kTcFold = 32;      // TMEM groups (64 rows each) per fp64 fold

// ------------------------------------------------------------ tcgen05 PTX ---
// shared-memory matrix descriptor, no swizzle.  MN-major canonical layout:
// a core matrix is 8 K-rows x 16 bytes (4 tf32 along M/N), 128 B contiguous;
// LBO = byte stride between core matrices along K, SBO = along M/N.
__host__ __device__ constexpr uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1 (sm_100)
}
// instruction descriptor: D f32, A/B tf32, M x N; mn = 1: both operands
// MN-major (bits 15, 16), else K-major
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, int mn = 0) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

// two 16-column TMEM loads (leading-product and cross-term accumulators)
// behind a single wait
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float *va, float *vb) {
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

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// round-to-nearest (ties away) to TF32 with integer ops: cvt.rna.tf32.f32
// runs on the quarter-rate conversion pipe, which limited the converters
__device__ __forceinline__ float tf32_round(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// x = p[0] + ... + p[NS-1] in TF32 pieces (the MMA reads the top 19 bits of
// each; the last piece is left unrounded and is truncated by the hardware)
template <int NS>
__device__ __forceinline__ void split_tf32(float x, float (&p)[3]) {
  p[0] = tf32_round(x);
  const float r = x - p[0];
  if (NS == 3) {
    p[1] = tf32_round(r);
    p[2] = r - p[1];
  } else {
    p[1] = r;
  }
}

// tile configuration: NS pieces, TK rows per operand stage, FL stages per
// TMEM accumulation group.  Products kept: all (a, b) with a + b < NS plus,
// for NS = 3, (1, 1): error ~2^-24 (NS = 3) / 2^-21 (NS = 2) per product.
// TK rows per tile (2 MMA k-steps), RS raw stages in flight (~100 KB of
// outstanding bulk copies per SM to cover HBM latency), OS operand stages.
template <int NS>
struct TcCfg {
  static constexpr int TK = NS == 3 ? 16 : 32;
  static constexpr int FL = NS == 3 ? 4 : 2;
  static constexpr int RS = NS == 3 ? 8 : 3;
  static constexpr int OS = NS == 3 ? 2 : 2;
  static constexpr int MI = (112 + 2 * 56) * (TK / 4) / (kTcThreads - 64) + 1;  // items/thread
  static constexpr int NPROD = NS == 3 ? 6 : 3;
  __host__ __device__ static constexpr int pa(int t) { return t == 1 ? 1 : t == 3 ? 2 : t == 5 ? 1 : 0; }
  __host__ __device__ static constexpr int pb(int t) { return t == 2 ? 1 : t == 4 ? 2 : t == 5 ? 1 : 0; }
};

// ---------------------------------------------------------------- kernel ---
struct GramTcArgs {
  int64_t n;
  int ld, w;     // row stride, Gram width (w <= 112)
  int nh;        // columns per half (<= 64)
  int npairs;    // CTA pairs (grid = 2 * npairs)
  double *part;  // [grid][2][kTcM][kTcN], zeroed by the host; fp64 accumulation
  int dbg;       // MG_TC_DBG bits (timing experiments): 1 no MMA, 2 no convert, 4 no epilogue
};

// dynamic shared memory: raw ring (RS stages of S rows, AS rows, b), then the
// operand ring (OS stages of [A pieces | bS pieces | AS pieces]), then the
// mbarriers and the TMEM address slot
template <int NS>
__host__ __device__ inline size_t tc_raw_bytes(int ld) {
  return ((size_t)2 * TcCfg<NS>::TK * ld * 4 + 128 + 127) / 128 * 128;
}
template <int NS>
__host__ __device__ constexpr size_t tc_op_bytes() {
  return (size_t)NS * (kTcM + 2 * kTcN) * TcCfg<NS>::TK * 4;
}
template <int NS>
__host__ __device__ inline size_t tc_smem_bytes(int ld) {
  return TcCfg<NS>::RS * tc_raw_bytes<NS>(ld) + TcCfg<NS>::OS * tc_op_bytes<NS>() + 32 * 8 +
         16;  // mbarriers, TMEM slot
}

// TMEM per accumulation buffer (256 columns): [hi*hi G_B | hi*hi G_A |
// cross terms G_B | cross terms G_A].  The leading products and the small
// cross products accumulate separately, so the tensor core's fp32 adds round
// the cross terms against their own (2^-11 smaller) magnitude.
__device__ __forceinline__ void tc_drain(int fg, uint32_t tbase, int q, int g, int lane,
                                         uint64_t *tm_full, uint64_t *tm_empty,
                                         float (&acc)[kTcN], bool skip) {
  const int buf = fg & 1;
  mbar_wait(&tm_full[buf], (fg >> 1) & 1);
  __syncwarp();  // tcgen05.ld is warp-collective (.sync.aligned)
  tc_fence_after();
  const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + buf * 256 + g * 64;
#pragma unroll
  for (int c = 0; c < (skip ? 0 : kTcN); c += 16) {
    float v[16], x[16];
    tmem_ld16x2(ta + c, ta + 128 + c, v, x);
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[c + e] += v[e] + x[e];
  }
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&tm_empty[buf]);
}

// 10 warps, one role each:
//   warp 0      bulk-copy producer (lane 0): raw ring refills as soon as the
//               workers release a stage (raw_empty)
//   warp 1      MMA issuer (lane 0): waits op_full, issues the tcgen05.mma
//               stream of a tile, commits op_empty / tm_full
//   warps 2-9   workers: convert raw fp32 rows into TF32 pieces (fixed items
//               per thread), then drain their TMEM quadrant every 64 rows
//               into fp32 registers, folded into the fp64 CTA partial in
//               global memory every kTcFold groups
template <int NS>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_gram_tc(const float *__restrict__ S, const float *__restrict__ AS,
              const float *__restrict__ b, GramTcArgs a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  using C = TcCfg<NS>;
  constexpr int TK = C::TK, FL = C::FL, RS = C::RS, OS = C::OS;
  constexpr int NW = kTcThreads - 64;  // worker threads
  constexpr int NWW = NW / 32;         // worker warps
  const int ld = a.ld, w = a.w;
  const size_t RAW = tc_raw_bytes<NS>(ld), OP = tc_op_bytes<NS>();
  unsigned char *raw0 = sm, *op0 = sm + RS * RAW;
  uint64_t *bars = reinterpret_cast<uint64_t *>(op0 + OS * OP);
  uint64_t *raw_full = bars, *raw_empty = bars + RS, *op_full = bars + 2 * RS,
           *op_empty = op_full + OS, *tm_full = op_empty + OS, *tm_empty = tm_full + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 32);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x & 1, pair = blockIdx.x >> 1;
  const int c0 = h * a.nh;                      // first Gram column of this CTA
  const int ncol = max(0, min(a.nh, w - c0));   // valid columns of this half
  const int64_t ntiles = (a.n + TK - 1) / TK;
  const int64_t t_begin = ntiles * pair / a.npairs;
  const int64_t t_end = ntiles * (pair + 1) / a.npairs;
  const int T = (int)(t_end - t_begin);

  // zero the operand rings once: padded rows/columns are never written again
  {
    float4 *pa = reinterpret_cast<float4 *>(op0);
    const int n4 = (int)(OS * OP / 16);
    for (int e = tid; e < n4; e += kTcThreads) pa[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (tid == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], NWW);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(&op_full[s], NWW);
      mbar_init(&op_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], NWW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();  // zeroed operand tiles visible to the tensor core
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  auto raw_stage = [&](int s) { return reinterpret_cast<float *>(raw0 + (size_t)s * RAW); };

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    if (lane == 0)
      for (int t = 0; t < T; ++t) {
        const int s = t % RS;
        mbar_wait(&raw_empty[s], ((t / RS) & 1) ^ 1);
        float *rs = raw_stage(s);
        issue_tile<float>(S, (a.dbg & 64) ? nullptr : AS, (a.dbg & 32) ? nullptr : b, a.n, ld,
                          TK, t_begin + t, rs, rs + (size_t)TK * ld, rs + (size_t)2 * TK * ld,
                          &raw_full[s]);
      }
    __syncwarp();  // reconverge before the aligned CTA barrier below
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issue
    // K-major, no swizzle (see the worker layout); one MMA k-step (8 rows)
    // spans two core matrices along K
    constexpr uint32_t idesc = umma_idesc_tf32(kTcM, kTcN);
    constexpr uint32_t LBO_A = (kTcM / 8) * 128, LBO_B = (kTcN / 8) * 128, SBO = 128;
    constexpr uint32_t OPA = kTcM * TK * 4, OPB = kTcN * TK * 4;
    constexpr uint64_t dA0 = umma_desc(0, LBO_A, SBO), dB0 = umma_desc(0, LBO_B, SBO);
    const uint32_t op_base = smem_u32(op0);
    if (lane == 0)
      for (int t = 0; t < T; ++t) {
        const int so = t % OS;
        const int fg = t / FL, buf = fg & 1;
        const bool first = (t % FL) == 0;
        const bool last = (t % FL) == FL - 1 || t == T - 1;
        if (first) mbar_wait(&tm_empty[buf], ((fg >> 1) & 1) ^ 1);
        mbar_wait(&op_full[so], (t / OS) & 1);
        tc_fence_after();
        const uint32_t A = op_base + so * (uint32_t)OP, B = A + NS * OPA;
        const uint32_t dB = tbase + buf * 256, dA = dB + 64;
        if (!(a.dbg & 1)) {
#pragma unroll
          for (int k = 0; k < TK / 8; ++k) {
#pragma unroll
            for (int pr = 0; pr < C::NPROD; ++pr) {
              const int t2 = C::NPROD - 1 - pr;  // small products first
              const uint64_t da = dA0 | ((A + C::pa(t2) * OPA + k * 2 * LBO_A) >> 4);
              const uint64_t db = dB0 | ((B + C::pb(t2) * OPB + k * 2 * LBO_B) >> 4);
              const uint64_t dx = dB0 | ((B + (NS + C::pb(t2)) * OPB + k * 2 * LBO_B) >> 4);
              // leading product -> [0, 128), cross products -> [128, 256)
              const uint32_t off = t2 == 0 ? 0u : 128u;
              const bool init = first && k == 0 && (t2 == 0 || pr == 0);
              const uint32_t acc = init ? 0u : 1u;
              umma_tf32(dB + off, da, db, idesc, acc);
              umma_tf32(dA + off, da, dx, idesc, acc);
            }
          }
        }
        umma_commit(&op_empty[so]);
        if (last) umma_commit(&tm_full[buf]);
      }
    __syncwarp();  // lanes 1-31 must not reach the barrier / dealloc early
  } else {
    // ---------------------------------------------------------- workers
    const int wt = tid - 64;
    const int q = warp & 3;         // TMEM lane quadrant of this warp
    const int g = (warp - 2) >> 2;  // 0: G_B columns, 1: G_A columns
    // fixed conversion items of this thread: (column m, 4-row group kg) of A
    // (w columns), bS and AS (this half's columns).  Operand layout (K-major,
    // no swizzle): element (m, k) of a piece at byte (m / 8) * 128 + (m % 8)
    // * 16 + (k / 4) * LBO + (k % 4) * 4 -- core matrices of 8 columns x 16 B
    // of K, M-adjacent ones contiguous (SBO = 128 B), K-adjacent ones LBO =
    // M / 8 * 128 B apart.  An item loads rows 4kg..4kg+3 of one column and
    // stores one float4 per piece; a warp covers 32 consecutive columns
    // (conflict-free loads and stores).
    // my_src: byte offset of (row 4kg, column) in the raw stage | kg << 24;
    // my_dst: byte offset in the operand stage | bit 28 (B piece) | bit 31 (scale by b)
    const int nA = w * (TK / 4), nB = ncol * (TK / 4);
    int my_src[C::MI], my_dst[C::MI], my_n = 0;
#pragma unroll
    for (int u = 0; u < C::MI; ++u) {
      const int it = wt + u * NW;
      my_src[u] = my_dst[u] = 0;
      if (it < nA + 2 * nB) {
        int m, kg, kind;
        if (it < nA) {
          kind = 0;
          m = it % w;
          kg = it / w;
        } else {
          const int v = it - nA;
          kind = v < nB ? 1 : 2;
          const int r = v - (kind - 1) * nB;
          m = r % ncol;
          kg = r / ncol;
        }
        const int col = kind == 0 ? m : c0 + m;
        my_src[u] = (((kind == 2 ? TK * ld : 0) + 4 * kg * ld + col) * 4) | (kg << 24);
        const int lbo = (kind == 0 ? kTcM : kTcN) / 8 * 128;
        const int dof = (kind == 0 ? 0 : NS * kTcM * TK * 4 + (kind == 2 ? NS * kTcN * TK * 4 : 0)) +
                        (m >> 3) * 128 + (m & 7) * 16 + kg * lbo;
        my_dst[u] = dof | (kind != 0 ? (1 << 28) : 0) | (kind == 1 ? (int)0x80000000 : 0);
        my_n = u + 1;
      }
    }
    if (a.dbg & 2) my_n = 0;
    float acc[kTcN];
#pragma unroll
    for (int j = 0; j < kTcN; ++j) acc[j] = 0.f;
    const int i = q * 32 + lane;  // Gram row of this thread
    double *dpart = a.part + ((size_t)blockIdx.x * 2 + g) * kTcM * kTcN + (size_t)i * kTcN;
    int drained = 0;
    for (int t = 0; t < T; ++t) {
      const int s = t % RS, so = t % OS;
      mbar_wait(&raw_full[s], (t / RS) & 1);
      mbar_wait(&op_empty[so], ((t / OS) & 1) ^ 1);  // MMAs of tile t-OS are done
      float *rS = raw_stage(s);
      float *rb = rS + (size_t)2 * TK * ld;
      const int nr = (int)min((int64_t)TK, a.n - (t_begin + t) * TK);
      if (nr < TK) {  // last tile: zero the stale rows, then convert branch-free
        float *rA = rS + (size_t)TK * ld;
        for (int e = wt; e < (TK - nr) * ld; e += NW) {
          rS[(size_t)nr * ld + e] = 0.f;
          rA[(size_t)nr * ld + e] = 0.f;
        }
        for (int e = nr + wt; e < TK; e += NW) rb[e] = 0.f;
        asm volatile("bar.sync 1, %0;" ::"n"(NW) : "memory");
      }
      const char *rbase = reinterpret_cast<const char *>(rS);
      char *obase = reinterpret_cast<char *>(op0 + (size_t)so * OP);
      float xs[C::MI][4];
#pragma unroll
      for (int u = 0; u < C::MI; ++u) {  // all loads first (independent)
        if (u < my_n) {
          const float *src = reinterpret_cast<const float *>(rbase + (my_src[u] & 0xFFFFFF));
          const bool sb = my_dst[u] < 0;
          const int k0 = 4 * (my_src[u] >> 24);
#pragma unroll
          for (int e = 0; e < 4; ++e) xs[u][e] = src[e * ld] * (sb ? rb[k0 + e] : 1.f);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&raw_empty[s]);  // raw stage s no longer read
#pragma unroll
      for (int u = 0; u < C::MI; ++u) {
        if (u < my_n) {
          float pc[4][3];
#pragma unroll
          for (int e = 0; e < 4; ++e) split_tf32<NS>(xs[u][e], pc[e]);
          const int d = my_dst[u] & 0x7FFFFFFF;
          const int pstride = (d >> 28) ? kTcN * TK * 4 : kTcM * TK * 4;  // bytes
          char *dst = obase + (d & 0x0FFFFFFF);
#pragma unroll
          for (int p = 0; p < NS; ++p)
            *reinterpret_cast<float4 *>(dst + p * pstride) =
                make_float4(pc[0][p], pc[1][p], pc[2][p], pc[3][p]);
        }
      }
      fence_proxy_async();  // generic-proxy operand writes -> async proxy (MMA)
      __syncwarp();
      if (lane == 0) mbar_arrive(&op_full[so]);
      // drain group g half a group after it closed: the MMAs have had time to
      // finish, and group g+2 (same TMEM buffer) starts only later
      if (t >= FL + FL / 2 && (t - FL / 2) % FL == 0) {
        tc_drain(drained++, tbase, q, g, lane, tm_full, tm_empty, acc, a.dbg & 4);
        if (drained % kTcFold == 0) {  // fp32 group sums -> fp64 CTA partial
#pragma unroll
          for (int j = 0; j < kTcN; ++j) {
            dpart[j] += (double)acc[j];
            acc[j] = 0.f;
          }
        }
      }
    }
    for (const int ng = (T + FL - 1) / FL; drained < ng;)
      tc_drain(drained++, tbase, q, g, lane, tm_full, tm_empty, acc, a.dbg & 4);
    if (a.dbg & 8) {
      float sacc = 0.f;
      for (int j = 0; j < kTcN; ++j) sacc += acc[j];
      dpart[0] = 1000.0 + T;
      dpart[1] = drained;
      dpart[2] = sacc;
      dpart[3] = my_n;
      dpart[4] = tbase;
    } else {
#pragma unroll
      for (int j = 0; j < kTcN; ++j) dpart[j] += (double)acc[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

// sum the pair partials (fixed order).  Mirror convention of k_reduce_gram2:
// entries in block-lower 8x8 blocks come from the block-upper product, so
// G_A[i][j] (i < j) = S_i' (AS)_j uses the freshly multiplied A-image of the
// later column (AW from the SpMM, not the carried AX / AP).
__global__ void k_reduce_gram_tc(const double *__restrict__ part, int npairs, int w, int nh,
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
    const int h = j >= nh ? 1 : 0, jl = j - h * nh;
    double s = 0.0;
    for (int c = 0; c < npairs; ++c)
      s += part[(((size_t)(2 * c + h) * 2 + g) * kTcM + i) * kTcN + jl];
    (g ? GA : GB)[r] = s;
  }
}

// ------------------------------------------------------ update (tcgen05) ---
// P = S Zp, X = S Zx (Zx = Zp + [Yx; 0; 0]) and the same for AS, as one
// tensor-core GEMM per matrix: D[128 rows x 80] = S[rows, 0:K] * [Zp | Zx]
// with 3xTF32 pieces; then the residual block W = prec (AX - b X theta), its
// column norms, and the write-back of [X P W] / [AX AP] / Wc.
//   A operand: S / AS row tiles (K-major, converted from row-major float4
//   loads, 32 K per stage); B operand: [Zp | Zx] pieces resident in smem.
static constexpr int kUpM = 128;      // rows per tile (MMA M)
static constexpr int kUpN = 80;       // [P | X] columns (2 * mp <= 80), zero-padded
// K per stage: 32 with 2 pieces, 16 with 3 (operand shared memory)
template <int NP>
struct UpCfg {
  static constexpr int KC = NP == 3 ? 16 : 32;
};
static constexpr int kUpKmax = 112;   // w <= 112
static constexpr int kUpThreads = 256;

struct UpdTcArgs {
  int64_t n;
  int ld, w, m, mp;
  const int *skip;   // device flag: nonzero -> return (fallback iteration)
  double *part;      // [grid][2*mp] column partials (rn^2, x^2)
  float *wc;         // compact W (n x mp)
};

__host__ __device__ constexpr size_t up_b_piece() { return (size_t)kUpN * kUpKmax * 4; }
template <int NP>
__host__ __device__ constexpr size_t up_a_piece() { return (size_t)kUpM * UpCfg<NP>::KC * 4; }
template <int NP>
__host__ __device__ constexpr size_t up_smem() {
  return NP * up_b_piece() + 2 * 2 * NP * up_a_piece<NP>() + 64 * 4 + 16 * 8 + 16;
}

__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float *v) {
  uint32_t r0, r1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  v[0] = __uint_as_float(r0);
  v[1] = __uint_as_float(r1);
}

template <int NP>
__global__ void __launch_bounds__(kUpThreads, 1)
    k_update_tc(float *__restrict__ S, float *__restrict__ AS, const float *__restrict__ b,
                const float *__restrict__ prec, const float *__restrict__ Mg,
                const double *__restrict__ theta, UpdTcArgs a) {
  if (*a.skip) return;
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int kUpKC = UpCfg<NP>::KC;
  constexpr size_t APC = up_a_piece<NP>();
  unsigned char *zb = sm;                           // [Zp|Zx] NP pieces (K-major, N=80 x K=112)
  unsigned char *st0 = sm + NP * up_b_piece();      // 2 stages x [S pieces, AS pieces]
  float *sth = reinterpret_cast<float *>(st0 + 2 * 2 * NP * APC);  // theta (mp <= 40)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sth + 64);
  uint64_t *st_empty = bars, *tm_full = bars + 2, *tm_empty = bars + 4;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ld = a.ld, w = a.w, mp = a.mp, m = a.m;
  constexpr uint32_t LBO_A = (kUpM / 8) * 128, LBO_B = (kUpN / 8) * 128, SBO = 128;

  // B operand: element (n, k) at (n/8)*128 + (n%8)*16 + (k/4)*LBO_B + (k%4)*4
  //   n < mp: Zp[k][n];  mp <= n < 2mp: Zx[k][n-mp] = Zp[k][n-mp] + (k < mp ? Yx[k][n-mp] : 0)
  for (int e = tid; e < kUpN * kUpKmax; e += kUpThreads) {
    const int n = e % kUpN, k = e / kUpN;
    float v = 0.f;
    if (k < w) {
      if (n < mp) v = Mg[k * mp + n];
      else if (n < 2 * mp) {
        const int c = n - mp;
        v = Mg[k * mp + c] + (k < mp ? Mg[w * mp + k * mp + c] : 0.f);
      }
    }
    float p[3];
    split_tf32<NP>(v, p);
    const int off = ((n >> 3) * 128 + (n & 7) * 16 + (k >> 2) * LBO_B + (k & 3) * 4) >> 2;
#pragma unroll
    for (int q = 0; q < NP; ++q) reinterpret_cast<float *>(zb + q * up_b_piece())[off] = p[q];
  }
  for (int e = tid; e < 64; e += kUpThreads) sth[e] = e < m ? (float)theta[e] : 0.f;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&st_empty[s], 1);
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], kUpThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  const int64_t ntiles = (a.n + kUpM - 1) / kUpM;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int T = (int)(t_end - t_begin);
  const int nkc = (w + kUpKC - 1) / kUpKC;  // K stages per tile
  // conversion mapping: lane -> (row r8 = lane % 8 within an 8-row group,
  // 16-byte K chunk c4 = lane / 8 + 4 * half); a warp loads 8 rows x 64 B
  const int q = warp & 3, half = warp >> 2;
  float sr[18], sx[18];
#pragma unroll
  for (int j = 0; j < 18; ++j) sr[j] = sx[j] = 0.f;

  // one K stage = 128 rows x kUpKC columns of S and AS: CPR 16-byte chunks
  // per row, J per thread; item e = tid + 256 j -> (row e / CPR, chunk e % CPR)
  constexpr int CPR = kUpKC / 4, J = kUpM * CPR / kUpThreads;
  float4 ld_s[J], ld_a[J];
  auto load_stage = [&](int64_t row0, int kc) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int e = tid + kUpThreads * j, r = e / CPR, c4 = e % CPR;
      const int col = kc * kUpKC + c4 * 4;
      const int64_t row = row0 + r;
      float4 vs = make_float4(0.f, 0.f, 0.f, 0.f), va = vs;
      if (row < a.n && col < ld) {
        vs = __ldg(reinterpret_cast<const float4 *>(S + row * ld + col));
        va = __ldg(reinterpret_cast<const float4 *>(AS + row * ld + col));
      }
      ld_s[j] = vs;
      ld_a[j] = va;
    }
  };
  auto store_stage = [&](int st) {
    unsigned char *base = st0 + (size_t)st * 2 * NP * APC;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int e = tid + kUpThreads * j, r = e / CPR, c4 = e % CPR;
      const int off = (r >> 3) * 128 + (r & 7) * 16 + c4 * LBO_A;
      float ps[4][3], pa[4][3];
      split_tf32<NP>(ld_s[j].x, ps[0]);
      split_tf32<NP>(ld_s[j].y, ps[1]);
      split_tf32<NP>(ld_s[j].z, ps[2]);
      split_tf32<NP>(ld_s[j].w, ps[3]);
      split_tf32<NP>(ld_a[j].x, pa[0]);
      split_tf32<NP>(ld_a[j].y, pa[1]);
      split_tf32<NP>(ld_a[j].z, pa[2]);
      split_tf32<NP>(ld_a[j].w, pa[3]);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        *reinterpret_cast<float4 *>(base + q * APC + off) =
            make_float4(ps[0][q], ps[1][q], ps[2][q], ps[3][q]);
        *reinterpret_cast<float4 *>(base + (NP + q) * APC + off) =
            make_float4(pa[0][q], pa[1][q], pa[2][q], pa[3][q]);
      }
    }
  };
  // epilogue of tile tt (TMEM buffer buf): thread = (row q*32+lane, 18 columns)
  auto epilogue = [&](int64_t tt, int buf, int use) {
    mbar_wait(&tm_full[buf], use & 1);
    __syncwarp();
    tc_fence_after();
    const int c0 = half * 18;
    const int64_t row = tt * kUpM + q * 32 + lane;
    const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + buf * 256;
    float P[18], X[18], AP[18], AX[18];
    tmem_ld16(ta + c0, P);
    tmem_ld2(ta + c0 + 16, P + 16);
    tmem_ld16(ta + mp + c0, X);
    tmem_ld2(ta + mp + c0 + 16, X + 16);
    // A-images: leading products (+80) and cross terms (+160) accumulate in
    // separate TMEM columns (the carried AX / AP are the drift-sensitive side)
    {
      float t1[18], t2[18];
      tmem_ld16(ta + 80 + c0, t1);
      tmem_ld2(ta + 80 + c0 + 16, t1 + 16);
      tmem_ld16(ta + 160 + c0, t2);
      tmem_ld2(ta + 160 + c0 + 16, t2 + 16);
#pragma unroll
      for (int j = 0; j < 18; ++j) AP[j] = t1[j] + t2[j];
      tmem_ld16(ta + 80 + mp + c0, t1);
      tmem_ld2(ta + 80 + mp + c0 + 16, t1 + 16);
      tmem_ld16(ta + 160 + mp + c0, t2);
      tmem_ld2(ta + 160 + mp + c0 + 16, t2 + 16);
#pragma unroll
      for (int j = 0; j < 18; ++j) AX[j] = t1[j] + t2[j];
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tm_empty[buf]);
    if (row < a.n) {
      const float br = b[row], pr = prec ? prec[row] : 1.f;
      float W[18];
#pragma unroll
      for (int j = 0; j < 18; ++j) {
        const int c = c0 + j;
        W[j] = 0.f;
        if (c < m) {
          const float r = AX[j] - br * X[j] * sth[c];
          sr[j] += r * r;
          sx[j] += X[j] * X[j];
          W[j] = pr * r;
        }
        if (c >= mp) X[j] = P[j] = W[j] = AX[j] = AP[j] = 0.f;
      }
      float *srow = S + row * ld, *arow = AS + row * ld, *wrow = a.wc + row * mp;
#pragma unroll
      for (int j = 0; j < 18; j += 2) {
        const int c = c0 + j;
        if (c < mp) {
          *reinterpret_cast<float2 *>(srow + c) = make_float2(X[j], X[j + 1]);
          *reinterpret_cast<float2 *>(srow + mp + c) = make_float2(P[j], P[j + 1]);
          *reinterpret_cast<float2 *>(srow + 2 * mp + c) = make_float2(W[j], W[j + 1]);
          *reinterpret_cast<float2 *>(arow + c) = make_float2(AX[j], AX[j + 1]);
          *reinterpret_cast<float2 *>(arow + mp + c) = make_float2(AP[j], AP[j + 1]);
          *reinterpret_cast<float2 *>(wrow + c) = make_float2(W[j], W[j + 1]);
        }
      }
    }
  };

  constexpr uint32_t idesc = umma_idesc_tf32(kUpM, kUpN);
  const uint64_t dA0 = umma_desc(0, LBO_A, SBO), dB0 = umma_desc(0, LBO_B, SBO);
  const uint32_t zb_base = smem_u32(zb), st_base = smem_u32(st0);
  int chunk = 0;  // global stage counter
  if (T > 0) load_stage(t_begin * kUpM, 0);
  for (int ti = 0; ti < T; ++ti) {
    const int64_t tt = t_begin + ti;
    const int buf = ti & 1;
    for (int kc = 0; kc < nkc; ++kc, ++chunk) {
      const int st = chunk & 1;
      mbar_wait(&st_empty[st], ((chunk >> 1) & 1) ^ 1);  // MMAs of chunk-2 done
      store_stage(st);
      // prefetch the next stage (next K chunk, or chunk 0 of the next tile)
      if (kc + 1 < nkc) load_stage(tt * kUpM, kc + 1);
      else if (ti + 1 < T) load_stage((tt + 1) * kUpM, 0);
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        if (kc == 0) mbar_wait(&tm_empty[buf], ((ti >> 1) & 1) ^ 1);
        tc_fence_after();
        const int ksteps = min(kUpKC, w - kc * kUpKC + 7) / 8;  // 8-row K steps in this stage
        const uint32_t A = st_base + st * 2 * NP * (uint32_t)APC;
        const uint32_t dS = tbase + buf * 256, dA = dS + 80, dA2 = dS + 160;
        for (int s = 0; s < ksteps; ++s) {
          const uint32_t kb = (uint32_t)(kc * (kUpKC / 4) + 2 * s) * LBO_B;  // B: K offset
          const uint32_t ka = 2 * s * LBO_A;
          uint64_t bq[NP], sq[NP], aq[NP];
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            bq[q] = dB0 | ((zb_base + q * (uint32_t)up_b_piece() + kb) >> 4);
            sq[q] = dA0 | ((A + q * (uint32_t)APC + ka) >> 4);
            aq[q] = dA0 | ((A + (NP + q) * (uint32_t)APC + ka) >> 4);
          }
          const uint32_t acc = (kc == 0 && s == 0) ? 0u : 1u;
          // small products first; NP = 3 keeps every (i, j) with i + j < 3 plus (1, 1)
          if (NP == 3) {
            umma_tf32(dS, sq[2], bq[0], idesc, acc);
            umma_tf32(dS, sq[0], bq[2], idesc, 1u);
            umma_tf32(dS, sq[1], bq[1], idesc, 1u);
            umma_tf32(dS, sq[1], bq[0], idesc, 1u);
            umma_tf32(dS, sq[0], bq[1], idesc, 1u);
            umma_tf32(dS, sq[0], bq[0], idesc, 1u);
            umma_tf32(dA2, aq[2], bq[0], idesc, acc);
            umma_tf32(dA2, aq[0], bq[2], idesc, 1u);
            umma_tf32(dA2, aq[1], bq[1], idesc, 1u);
            umma_tf32(dA2, aq[1], bq[0], idesc, 1u);
            umma_tf32(dA2, aq[0], bq[1], idesc, 1u);
            umma_tf32(dA, aq[0], bq[0], idesc, acc);
          } else {
            umma_tf32(dS, sq[1], bq[0], idesc, acc);
            umma_tf32(dS, sq[0], bq[1], idesc, 1u);
            umma_tf32(dS, sq[0], bq[0], idesc, 1u);
            umma_tf32(dA2, aq[1], bq[0], idesc, acc);
            umma_tf32(dA2, aq[0], bq[1], idesc, 1u);
            umma_tf32(dA, aq[0], bq[0], idesc, acc);
          }
        }
        umma_commit(&st_empty[st]);
        if (kc == nkc - 1) umma_commit(&tm_full[buf]);
      }
      __syncwarp();
      // drain the previous tile while this tile's MMAs run
      if (kc == 0 && ti > 0) epilogue(tt - 1, buf ^ 1, (ti - 1) >> 1);
    }
  }
  if (T > 0) epilogue(t_begin + T - 1, (T - 1) & 1, (T - 1) >> 1);
  // column partials: [rn^2 (mp) | x^2 (mp)] of this CTA, reduced over its rows
  tc_fence_before();
  __syncthreads();
  float *red = reinterpret_cast<float *>(st0);  // reuse the stage ring: [8 warps][2][18][32]
  {
#pragma unroll
    for (int j = 0; j < 18; ++j) {
      red[((warp * 2 + 0) * 18 + j) * 32 + lane] = sr[j];
      red[((warp * 2 + 1) * 18 + j) * 32 + lane] = sx[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < 2 * mp; c += kUpThreads) {
    const int which = c / mp, col = c - which * mp, hf = col / 18, j = col - hf * 18;
    double s = 0.0;
    for (int wq = 0; wq < 4; ++wq)
      for (int l = 0; l < 32; ++l) s += red[(((hf * 4 + wq) * 2 + which) * 18 + j) * 32 + l];
    a.part[(size_t)blockIdx.x * 2 * mp + c] = s;
  }
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

// Off by default (MG_TC_UPD=1 enables it): the 2-piece split carries ~2^-22
// relative error per product and the accumulation is not round-to-nearest,
// so the carried X / AX drift ~1e-5 per step against the CUDA-core update's
// ~1e-6 -- at C5 scale that costs 40-130% more LOBPCG iterations than it
// saves per iteration (profiles/r1_tc_update.md).
bool update_tc_supported(int w, int mp) {
  const char *e = getenv("MG_TC_UPD");
  if (!(e && e[0] == '1')) return false;
  return gram_tc_supported(w) && 2 * mp <= kUpN && mp <= 40 && w <= kUpKmax;
}

int update_tc(mg_ctx *ctx, int64_t n, int ld, int w, int m, int mp, float *S, float *AS,
              const float *b, const float *prec, const float *M, const double *theta,
              const int *skip, double *part, float *wc) {
  UpdTcArgs a{};
  a.n = n;
  a.ld = ld;
  a.w = w;
  a.m = m;
  a.mp = mp;
  a.skip = skip;
  a.part = part;
  a.wc = wc;
  const int64_t ntiles = (n + kUpM - 1) / kUpM;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms));
  static const int np = [] {
    const char *e = getenv("MG_TC_UPD_PIECES");
    return (e && e[0] == '2') ? 2 : 3;
  }();
  static thread_local bool attr = false;
  if (!attr) {
    MG_CUDA(cudaFuncSetAttribute(k_update_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)up_smem<2>()));
    MG_CUDA(cudaFuncSetAttribute(k_update_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)up_smem<3>()));
    attr = true;
  }
  if (np == 3)
    k_update_tc<3><<<grid, kUpThreads, up_smem<3>(), ctx->stream>>>(S, AS, b, prec, M, theta, a);
  else
    k_update_tc<2><<<grid, kUpThreads, up_smem<2>(), ctx->stream>>>(S, AS, b, prec, M, theta, a);
  MG_CHECK_LAUNCH(ctx);
  return grid;
}

template __global__ void k_gram_tc<2>(const float *, const float *, const float *, GramTcArgs);
template __global__ void k_gram_tc<3>(const float *, const float *, const float *, GramTcArgs);

static int tc_pieces() {
  const char *e = getenv("MG_TC_PIECES");
  return (e && e[0] == '3') ? 3 : 2;
}

bool gram_tc_supported(int w) {
  const char *e = getenv("MG_TC");
  if (e && e[0] == '0') return false;
  // v2 (mg_tc2.cu, the default) covers 48 < w <= 128; below that the CUDA-core
  // k_gram2 is faster (the per-tile pipeline cost of v2 dominates small tiles).
  // v1 (MG_TC_V=1 / MG_TC_PIECES=3): converter capacity limits it to 64 < w <= 112.
  return w > 48 && w <= 128 && w % 4 == 0;
}

void gram_pair_tc(mg_ctx *ctx, int64_t n, int ld, int w, const float *S, const float *AS,
                  const float *b, double *GB, double *GA, DBuf<double> &part) {
  require(ld % 4 == 0, MG_ERR_INTERNAL, "tc Gram: row stride must be a multiple of 4");
  const int NS = tc_pieces();
  {
    const char *e = getenv("MG_TC_V");  // 1: the v1 converter kernel
    if (NS == 2 && !(e && e[0] == '1') && gram_tc2_supported(w, ld)) {
      gram_pair_tc2(ctx, n, ld, w, S, AS, b, GB, GA, part);
      return;
    }
  }
  require(w > 64 && w <= 112 && w % 4 == 0, MG_ERR_INTERNAL, "tc Gram v1: needs 64 < w <= 112");
  const int TK = NS == 3 ? TcCfg<3>::TK : TcCfg<2>::TK;
  const int64_t ntiles = (n + TK - 1) / TK;
  const int npairs = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms / 2));
  const size_t need = (size_t)2 * npairs * 2 * kTcM * kTcN;
  if (part.n < need) part.alloc(ctx, need);
  GramTcArgs a{};
  a.n = n;
  a.ld = ld;
  a.w = w;
  a.nh = (w / 4 + 1) / 2 * 4;  // first half gets the odd 4-column group
  a.npairs = npairs;
  a.part = part.p;
  MG_CUDA(cudaMemsetAsync(part.p, 0, need * sizeof(double), ctx->stream));
  {
    const char *e = getenv("MG_TC_DBG");
    a.dbg = e ? atoi(e) : 0;
  }
  const size_t smem = NS == 3 ? tc_smem_bytes<3>(ld) : tc_smem_bytes<2>(ld);
  require(smem <= 227 * 1024, MG_ERR_INTERNAL, "tc Gram: row stride too large");
  static thread_local size_t smem_set[4] = {0, 0, 0, 0};
  if (smem > smem_set[NS]) {
    if (NS == 3)
      MG_CUDA(cudaFuncSetAttribute(k_gram_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    else
      MG_CUDA(cudaFuncSetAttribute(k_gram_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    smem_set[NS] = smem;
  }
  {
    ProfScope ps(ctx, PROF_GRAM, 2.0 * n * ld * sizeof(float));
    if (NS == 3)
      k_gram_tc<3><<<2 * npairs, kTcThreads, smem, ctx->stream>>>(S, AS, b, a);
    else
      k_gram_tc<2><<<2 * npairs, kTcThreads, smem, ctx->stream>>>(S, AS, b, a);
    MG_CHECK_LAUNCH(ctx);
  }
  k_reduce_gram_tc<<<grid_for(2 * w * w, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
      part.p, npairs, w, a.nh, GB, GA);
  MG_CHECK_LAUNCH(ctx);
}

}  // namespace mg
