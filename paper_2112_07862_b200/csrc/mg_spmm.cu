// Staged SpMM: Y = A X for the narrow blocks of the LOBPCG loop (A W, 16..36
// fp32 columns), with the gathered rows of X held in shared memory.
//
// Status: opt-in (MG_SPMM_STAGED=1), see build_blocked.
// Why (profiles/r1_spmm.md): the row-per-sub-warp k_spmm gathers one 144-byte
// row of X per nonzero through L1; with the Cuthill-McKee order ~68 % of those
// hit, but the L1/TEX pipe (77 % busy) and the L2 misses of the rest bound it
// at ~1 TB/s of algorithmic traffic.  Here each CTA owns a block of kRB rows:
//   1. the block's distinct columns (precomputed once per matrix: sorted list
//      + a 16-bit local index per nonzero) are copied row by row into shared
//      memory with cp.async -- each needed row of X crosses L2 -> SM once per
//      block instead of once per nonzero (~9 distinct rows per block row at
//      C5 vs 37 nonzeros per row);
//   2. the rows are then formed from shared memory (LDS.128) with the same
//      sub-warp layout as k_spmm, reading 6 bytes per nonzero (u16 + fp32)
//      instead of 8.
// Blocks whose distinct-column set does not fit the shared-memory budget
// (or could not be indexed) use direct global gathers in the same kernel.
#include "mg_block.cuh"

namespace mg {

namespace {

constexpr int kRB = 32;           // rows per block
constexpr int kSortCap = 4096;    // max nonzeros per block that the builder indexes
constexpr int kBuildThreads = 256;
constexpr int kStagedMaxW = 36;   // fp32 columns (one LOBPCG block at K = 32)
constexpr size_t kStageBudget = 54 * 1024;  // four CTAs per SM

// one CTA per row block: sort the block's column ids, count (mode 0) or write
// (mode 1) the distinct ones and the local index of every nonzero
template <int MODE>
__global__ void __launch_bounds__(kBuildThreads)
    k_blk_build(int64_t n, const int64_t *__restrict__ ptr, const int *__restrict__ idx,
                int64_t *__restrict__ cnt, const int64_t *__restrict__ uoff, int *__restrict__ ucol,
                uint16_t *__restrict__ lidx) {
  __shared__ int key[kSortCap];
  __shared__ int scan[kBuildThreads + 1];
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * kRB, r1 = min(n, r0 + kRB);
  const int64_t k0 = ptr[r0], E64 = ptr[r1] - k0;
  const int tid = threadIdx.x;
  if (E64 > kSortCap || E64 == 0) {
    if (MODE == 0 && tid == 0) cnt[b] = 0;
    return;
  }
  const int E = (int)E64;
  int P = 1;
  while (P < E) P <<= 1;
  for (int e = tid; e < P; e += kBuildThreads) key[e] = e < E ? idx[k0 + e] : 0x7fffffff;
  __syncthreads();
  // bitonic sort of P keys
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = tid; e < P / 2; e += kBuildThreads) {
        const int lo = 2 * e - (e & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const int a = key[lo], c = key[hi];
        if ((a > c) == up) {
          key[lo] = c;
          key[hi] = a;
        }
      }
      __syncthreads();
    }
  // distinct flags -> per-thread counts over contiguous ranges -> scan
  const int per = (E + kBuildThreads - 1) / kBuildThreads;
  const int e0 = tid * per, e1 = min(E, e0 + per);
  int c = 0;
  for (int e = e0; e < e1; ++e) c += (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
  scan[tid + 1] = c;
  if (tid == 0) scan[0] = 0;
  __syncthreads();
  if (tid == 0)
    for (int q = 1; q <= kBuildThreads; ++q) scan[q] += scan[q - 1];
  __syncthreads();
  const int U = scan[kBuildThreads];
  if (MODE == 0) {
    if (tid == 0) cnt[b] = U > 65535 ? 0 : U;
    return;
  }
  if (uoff[b + 1] - uoff[b] != U) return;  // block left unindexed by the count pass
  int *uc = ucol + uoff[b];
  int rk = scan[tid];
  for (int e = e0; e < e1; ++e)
    if (e == 0 || key[e] != key[e - 1]) uc[rk++] = key[e];
  __syncthreads();
  // local index of every nonzero: binary search in the (global) distinct list
  for (int e = tid; e < E; e += kBuildThreads) {
    const int col = idx[k0 + e];
    int lo = 0, hi = U - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (uc[mid] < col) lo = mid + 1;
      else hi = mid;
    }
    lidx[k0 + e] = (uint16_t)lo;
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

template <typename T, bool DIFF>
__global__ void __launch_bounds__(256)
    k_spmm_st(int64_t n, const int64_t *__restrict__ ptr, const int *__restrict__ idx,
              const T *__restrict__ val, const int64_t *__restrict__ uoff,
              const int *__restrict__ ucol, const uint16_t *__restrict__ lidx,
              const T *__restrict__ X, int ldx, T *__restrict__ Y, int ldy, int w, int cap,
              const T *__restrict__ rowsum) {
  using V = typename VecT<T>::V;
  constexpr int VN = VecT<T>::N;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sX = reinterpret_cast<T *>(sm_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = w / VN, G = 32 / L;
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * kRB, r1 = min(n, r0 + kRB);
  const int64_t u0 = uoff[b];
  const int U = (int)(uoff[b + 1] - u0);
  const bool staged = U > 0 && U <= cap;
  if (staged) {
    const int C = L;  // 16-byte chunks per row
    for (int e = tid; e < U * C; e += 256) {
      const int u = e / C, c = e - u * C;
      cp_async16(sX + (size_t)u * w + c * VN, X + (int64_t)ucol[u0 + u] * ldx + c * VN);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  const int g = lane / L, gl = lane - g * L;
  if (g >= G) return;
  for (int64_t row = r0 + warp * G + g; row < r1; row += 8 * G) {
    const int64_t s = ptr[row], e = ptr[row + 1];
    T acc[VN], xi[VN];
#pragma unroll
    for (int q = 0; q < VN; ++q) acc[q] = T(0), xi[q] = T(0);
    if (DIFF) {
      const V xs = reinterpret_cast<const V *>(X + row * (int64_t)ldx)[gl];
      const T *ps = reinterpret_cast<const T *>(&xs);
#pragma unroll
      for (int q = 0; q < VN; ++q) xi[q] = ps[q];
    }
    int64_t k = s;
    if (staged) {
      for (; k + 4 <= e; k += 4) {
        const int j0 = lidx[k], j1 = lidx[k + 1], j2 = lidx[k + 2], j3 = lidx[k + 3];
        const T v0 = val[k], v1 = val[k + 1], v2 = val[k + 2], v3 = val[k + 3];
        const V x0 = reinterpret_cast<const V *>(sX + (size_t)j0 * w)[gl];
        const V x1 = reinterpret_cast<const V *>(sX + (size_t)j1 * w)[gl];
        const V x2 = reinterpret_cast<const V *>(sX + (size_t)j2 * w)[gl];
        const V x3 = reinterpret_cast<const V *>(sX + (size_t)j3 * w)[gl];
        const T *p0 = reinterpret_cast<const T *>(&x0), *p1 = reinterpret_cast<const T *>(&x1),
                *p2 = reinterpret_cast<const T *>(&x2), *p3 = reinterpret_cast<const T *>(&x3);
#pragma unroll
        for (int q = 0; q < VN; ++q) {
          acc[q] += DIFF ? v0 * (p0[q] - xi[q]) : v0 * p0[q];
          acc[q] += DIFF ? v1 * (p1[q] - xi[q]) : v1 * p1[q];
          acc[q] += DIFF ? v2 * (p2[q] - xi[q]) : v2 * p2[q];
          acc[q] += DIFF ? v3 * (p3[q] - xi[q]) : v3 * p3[q];
        }
      }
      for (; k < e; ++k) {
        const V x0 = reinterpret_cast<const V *>(sX + (size_t)lidx[k] * w)[gl];
        const T v0 = val[k];
        const T *p0 = reinterpret_cast<const T *>(&x0);
#pragma unroll
        for (int q = 0; q < VN; ++q) acc[q] += DIFF ? v0 * (p0[q] - xi[q]) : v0 * p0[q];
      }
    } else {
      for (; k < e; ++k) {
        const V x0 = reinterpret_cast<const V *>(X + (int64_t)idx[k] * ldx)[gl];
        const T v0 = val[k];
        const T *p0 = reinterpret_cast<const T *>(&x0);
#pragma unroll
        for (int q = 0; q < VN; ++q) acc[q] += DIFF ? v0 * (p0[q] - xi[q]) : v0 * p0[q];
      }
    }
    if (DIFF) {
      const T rs = rowsum[row];
#pragma unroll
      for (int q = 0; q < VN; ++q) acc[q] += rs * xi[q];
    }
    V out;
    T *po = reinterpret_cast<T *>(&out);
#pragma unroll
    for (int q = 0; q < VN; ++q) po[q] = acc[q];
    reinterpret_cast<V *>(Y + row * ldy)[gl] = out;
  }
}

}  // namespace

template <typename T>
void build_blocked(mg_ctx *ctx, OwnedCSR<T> &A) {
  const int64_t n = A.view.n, nnz = A.view.nnz;
  // opt-in (MG_SPMM_STAGED=1): with the Cuthill-McKee order a 32-row block
  // still touches ~12 distinct rows of X per row, and staging them lost to
  // k_spmm's L1 hits (profiles/r1_spmm.md: 1.10 vs 0.96 ms at C5 2M); it pays
  // only with a more compact node order
  const char *env = getenv("MG_SPMM_STAGED");
  if (!(env && env[0] == '1') || n < 4 * kRB || nnz < 8 * n) return;
  const int64_t nblk = (n + kRB - 1) / kRB;
  DBuf<int64_t> cnt(ctx, nblk);
  A.uoff.alloc(ctx, nblk + 1);
  k_blk_build<0><<<(unsigned)nblk, kBuildThreads, 0, ctx->stream>>>(n, A.view.ptr, A.view.idx,
                                                                   cnt.p, nullptr, nullptr, nullptr);
  MG_CHECK_LAUNCH(ctx);
  const int64_t tot = exclusive_scan_i64(ctx, cnt.p, A.uoff.p, nblk);
  A.ucol.alloc(ctx, tot > 0 ? tot : 1);
  A.lidx.alloc(ctx, nnz > 0 ? nnz : 1);
  k_blk_build<1><<<(unsigned)nblk, kBuildThreads, 0, ctx->stream>>>(
      n, A.view.ptr, A.view.idx, nullptr, A.uoff.p, A.ucol.p, A.lidx.p);
  MG_CHECK_LAUNCH(ctx);
  A.view.rb = kRB;
  A.view.nblk = nblk;
  A.view.uoff = A.uoff.p;
  A.view.ucol = A.ucol.p;
  A.view.lidx = A.lidx.p;
}

template <typename T>
bool spmm_staged(mg_ctx *ctx, const DevCSR<T> &A, const T *X, int ldx, T *Y, int ldy, int w) {
  constexpr int VN = VecT<T>::N;
  if (!A.lidx || A.rb != kRB || sizeof(T) != 4 || w < 4 * VN || w > kStagedMaxW || w % VN) return false;
  const int cap = (int)(kStageBudget / ((size_t)w * sizeof(T)));
  const size_t smem = (size_t)cap * w * sizeof(T);
  static thread_local size_t set = 0;
  if (smem > set) {
    MG_CUDA(cudaFuncSetAttribute(k_spmm_st<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kStageBudget));
    MG_CUDA(cudaFuncSetAttribute(k_spmm_st<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kStageBudget));
    set = kStageBudget;
  }
  if (A.rowsum)
    k_spmm_st<T, true><<<(unsigned)A.nblk, 256, smem, ctx->stream>>>(
        A.n, A.ptr, A.idx, A.val, A.uoff, A.ucol, A.lidx, X, ldx, Y, ldy, w, cap, A.rowsum);
  else
    k_spmm_st<T, false><<<(unsigned)A.nblk, 256, smem, ctx->stream>>>(
        A.n, A.ptr, A.idx, A.val, A.uoff, A.ucol, A.lidx, X, ldx, Y, ldy, w, cap, nullptr);
  MG_CHECK_LAUNCH(ctx);
  return true;
}

template void build_blocked<float>(mg_ctx *, OwnedCSR<float> &);
template void build_blocked<double>(mg_ctx *, OwnedCSR<double> &);
template bool spmm_staged<float>(mg_ctx *, const DevCSR<float> &, const float *, int, float *, int,
                                 int);
template bool spmm_staged<double>(mg_ctx *, const DevCSR<double> &, const double *, int, double *,
                                  int, int);

}  // namespace mg
