// numpy's Generator(PCG64).standard_normal stream on the device, bit for bit:
// the reference's initial block X0 = default_rng(seed).standard_normal((n, m))
// (eigensolver.py:177-178, 189).  At config 5 that is 660M normals, ~7 s of
// single-threaded numpy on the host before the solve can start.
//
//   PCG64 (PCG XSL-RR 128/64): s <- s * M + inc (mod 2^128), out = rotr64(hi ^ lo,
//     s >> 122); jump-ahead by d draws with the O(log d) LCG advance.
//   standard normal: 256-layer ziggurat (tables in mg_ziggurat_tables.h, read
//     back from the installed numpy by tools/gen_ziggurat_tables.py); a normal
//     takes one draw 99 % of the time, more on the slow / tail paths.
//
// Variable consumption makes the stream sequential; in parallel:
//   1. k_zig_scan: thread j walks draws [jB, jB + B) as if a normal started at
//      jB, recording which positions start a normal (bitmap) and where the
//      walk leaves the chunk;
//   2. host stitch: the true first start of chunk j is the exit of chunk j-1;
//      if the speculative walk passed through it (almost always: walks merge
//      as soon as one lands on the other's path) the chunk's starts are a
//      suffix of the bitmap, else the host re-walks that chunk;
//   3. k_zig_emit: thread j re-walks from its true entry and writes its normals
//      at the prefix-summed output offset.
// Tail draws (layer 0, ~1 in 2700) go through log1p; the host recomputes
// those few values with the C library's log1p (numpy's), so the stream is
// identical to numpy's, not just within an ulp.
#include <cmath>
#include <vector>

#include "mg_common.cuh"
#include "mg_rng.cuh"
#include "mg_ziggurat_tables.h"

namespace mg {

namespace {

typedef unsigned __int128 u128;
constexpr int kZigB = 4096;  // draws per chunk
constexpr u128 kPcgMult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

__constant__ uint64_t cKi[256];
__constant__ double cWi[256];
__constant__ double cFi[256];

__host__ __device__ inline u128 pcg_advance(u128 state, uint64_t delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

struct Pcg {
  u128 s, inc;
  __host__ __device__ inline uint64_t next() {
    s = s * kPcgMult + inc;
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __host__ __device__ inline double next_double() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// one standard normal; returns draws consumed; *tail = 1 if the value came
// from the tail (log1p) branch
template <bool DEV>
__host__ __device__ inline int zig_normal(Pcg &g, double &out, int &tail) {
  int used = 0;
  tail = 0;
  for (;;) {
    uint64_t r = g.next();
    ++used;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
#ifdef __CUDA_ARCH__
    const uint64_t ki = cKi[idx];
    const double wi = cWi[idx];
#else
    const uint64_t ki = kZigKiH[idx];
    const double wi = kZigWiH[idx];
#endif
    double x = (double)rabs * wi;
    if (sign) x = -x;
    if (rabs < ki) {
      out = x;
      return used;
    }
    if (idx == 0) {
      for (;;) {
        const double u1 = g.next_double(), u2 = g.next_double();
        used += 2;
        const double xx = -kZigInvR * log1p(-u1);
        const double yy = -log1p(-u2);
        if (yy + yy > xx * xx) {
          out = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
          tail = 1;
          return used;
        }
      }
    }
#ifdef __CUDA_ARCH__
    const double f0 = cFi[idx - 1], f1 = cFi[idx];
    const double u = g.next_double();
    ++used;
    if (__dadd_rn(__dmul_rn(__dsub_rn(f0, f1), u), f1) < exp(-0.5 * x * x)) {
#else
    const double f0 = kZigFiH[idx - 1], f1 = kZigFiH[idx];
    const double u = g.next_double();
    ++used;
    if ((f0 - f1) * u + f1 < std::exp(-0.5 * x * x)) {
#endif
      out = x;
      return used;
    }
  }
}

__global__ void k_zig_scan(u128 s0, u128 inc, int64_t nchunks, uint32_t *__restrict__ bits,
                           int64_t *__restrict__ exitp, int32_t *__restrict__ cnt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nchunks) return;
  const int64_t base = j * kZigB;
  Pcg g{pcg_advance(s0, (uint64_t)base, kPcgMult, inc), inc};
  uint32_t *bm = bits + j * (kZigB / 32);
  for (int w = 0; w < kZigB / 32; ++w) bm[w] = 0;
  int64_t p = base;
  int c = 0;
  while (p < base + kZigB) {
    const int o = (int)(p - base);
    bm[o >> 5] |= 1u << (o & 31);
    double v;
    int tail;
    p += zig_normal<true>(g, v, tail);
    ++c;
  }
  exitp[j] = p;
  cnt[j] = c;
}

__global__ void k_zig_emit(u128 s0, u128 inc, int64_t nchunks, const int64_t *__restrict__ entry,
                           const int64_t *__restrict__ off, int64_t count, double *__restrict__ out,
                           int64_t *__restrict__ tails, int32_t *__restrict__ ntail, int tail_cap) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nchunks) return;
  const int64_t end = (j + 1) * kZigB;
  int64_t p = entry[j], o = off[j];
  if (p >= end || o >= count) return;
  Pcg g{pcg_advance(s0, (uint64_t)p, kPcgMult, inc), inc};
  while (p < end && o < count) {
    double v;
    int tail;
    const int64_t p0 = p;
    p += zig_normal<true>(g, v, tail);
    out[o] = v;
    if (tail) {  // host fixes the value with the C library's log1p
      const int t = atomicAdd(ntail, 1);
      if (t < tail_cap) {
        tails[2 * t] = o;
        tails[2 * t + 1] = p0;
      }
    }
    ++o;
  }
}

__global__ void k_zig_scatter(int n, const int64_t *__restrict__ pos, const double *__restrict__ v,
                              double *__restrict__ out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    out[pos[t]] = v[t];
}

}  // namespace

void normal_stream(mg_ctx *ctx, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                   uint64_t inc_lo, int64_t count, double *out) {
  require(count >= 0, MG_ERR_INPUT, "normal stream: negative count");
  if (count == 0) return;
  static thread_local int tables_dev = -1;
  if (tables_dev != ctx->device) {
    MG_CUDA(cudaMemcpyToSymbolAsync(cKi, kZigKiH, sizeof(kZigKiH), 0, cudaMemcpyHostToDevice,
                                    ctx->stream));
    MG_CUDA(cudaMemcpyToSymbolAsync(cWi, kZigWiH, sizeof(kZigWiH), 0, cudaMemcpyHostToDevice,
                                    ctx->stream));
    MG_CUDA(cudaMemcpyToSymbolAsync(cFi, kZigFiH, sizeof(kZigFiH), 0, cudaMemcpyHostToDevice,
                                    ctx->stream));
    tables_dev = ctx->device;
  }
  const u128 s0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  // ~1.2 % of normals take more than one draw; size the scan with a margin and
  // extend it (rarely) until the stitched count covers `count`
  int64_t nchunks = (int64_t)((double)count * 1.02 / kZigB) + 2;
  for (int attempt = 0;; ++attempt) {
    DBuf<uint32_t> bits(ctx, (size_t)nchunks * (kZigB / 32));
    DBuf<int64_t> exitp(ctx, nchunks);
    DBuf<int32_t> cnt(ctx, nchunks);
    const int thr = 128;
    k_zig_scan<<<(unsigned)((nchunks + thr - 1) / thr), thr, 0, ctx->stream>>>(s0, inc, nchunks,
                                                                              bits.p, exitp.p,
                                                                              cnt.p);
    MG_CHECK_LAUNCH(ctx);
    std::vector<uint32_t> hb((size_t)nchunks * (kZigB / 32));
    std::vector<int64_t> hx(nchunks);
    std::vector<int32_t> hc(nchunks);
    d2h_sync(ctx, hb.data(), bits.p, hb.size() * sizeof(uint32_t));
    d2h_sync(ctx, hx.data(), exitp.p, hx.size() * sizeof(int64_t));
    d2h_sync(ctx, hc.data(), cnt.p, hc.size() * sizeof(int32_t));
    // stitch
    std::vector<int64_t> entry(nchunks), off(nchunks);
    int64_t e = 0, total = 0;
    for (int64_t j = 0; j < nchunks; ++j) {
      const int64_t base = j * kZigB, end = base + kZigB;
      entry[j] = e;
      off[j] = total;
      if (e >= end) continue;  // a normal spanned the whole chunk
      const int o = (int)(e - base);
      const uint32_t *bm = hb.data() + (size_t)j * (kZigB / 32);
      if (bm[o >> 5] & (1u << (o & 31))) {  // the speculative walk passes through e
        int before = 0;
        for (int w = 0; w < (o >> 5); ++w) before += __builtin_popcount(bm[w]);
        before += __builtin_popcount(bm[o >> 5] & ((1u << (o & 31)) - 1u));
        total += hc[j] - before;
        e = hx[j];
      } else {  // re-walk this chunk from its true entry on the host
        Pcg g{pcg_advance(s0, (uint64_t)e, kPcgMult, inc), inc};
        while (e < end) {
          double v;
          int tail;
          e += zig_normal<false>(g, v, tail);
          ++total;
        }
      }
    }
    if (total < count) {
      nchunks = nchunks + nchunks / 50 + 2;
      require(attempt < 8, MG_ERR_INTERNAL, "normal stream: scan did not converge");
      continue;
    }
    DBuf<int64_t> dentry(ctx, nchunks), doff(ctx, nchunks);
    h2d(ctx, dentry.p, entry.data(), nchunks * sizeof(int64_t));
    h2d(ctx, doff.p, off.data(), nchunks * sizeof(int64_t));
    const int tail_cap = (int)std::min<int64_t>(count / 256 + 1024, 1 << 26);
    DBuf<int64_t> tails(ctx, 2 * (size_t)tail_cap);
    DBuf<int32_t> ntail(ctx, 1);
    MG_CUDA(cudaMemsetAsync(ntail.p, 0, sizeof(int32_t), ctx->stream));
    k_zig_emit<<<(unsigned)((nchunks + thr - 1) / thr), thr, 0, ctx->stream>>>(
        s0, inc, nchunks, dentry.p, doff.p, count, out, tails.p, ntail.p, tail_cap);
    MG_CHECK_LAUNCH(ctx);
    int32_t nt = 0;
    d2h_sync(ctx, &nt, ntail.p, sizeof(int32_t));
    require(nt <= tail_cap, MG_ERR_INTERNAL, "normal stream: tail list overflow");
    if (nt > 0) {  // exact tail values with the host C library's log1p (numpy's)
      std::vector<int64_t> ht(2 * (size_t)nt);
      d2h_sync(ctx, ht.data(), tails.p, ht.size() * sizeof(int64_t));
      std::vector<double> vals(nt);
      for (int t = 0; t < nt; ++t) {
        Pcg g{pcg_advance(s0, (uint64_t)ht[2 * t + 1], kPcgMult, inc), inc};
        int tail;
        zig_normal<false>(g, vals[t], tail);
      }
      std::vector<int64_t> pos(nt);
      for (int t = 0; t < nt; ++t) pos[t] = ht[2 * t];
      DBuf<double> dv(ctx, nt);
      DBuf<int64_t> dp(ctx, nt);
      h2d(ctx, dv.p, vals.data(), nt * sizeof(double));
      h2d(ctx, dp.p, pos.data(), nt * sizeof(int64_t));
      k_zig_scatter<<<grid_for(nt, 256, 1024), 256, 0, ctx->stream>>>(nt, dp.p, dv.p, out);
      MG_CHECK_LAUNCH(ctx);
    }
    sync(ctx);
    return;
  }
}

}  // namespace mg
