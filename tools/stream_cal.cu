// calibration: streaming read bandwidth of LDG.128 vs cp.async.bulk rings
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
extern "C" __global__ void k_ldg(const float4 *x, long n4, float *out) {
  float4 a = make_float4(0, 0, 0, 0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = __ldg(x + i); a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  if (a.x == 12345.f) out[0] = a.y + a.z + a.w;
}
// ring of NS stages, each 'chunk' bytes, one producer thread, 8 consumer warps
extern "C" __global__ void k_bulk(const char *x, long bytes, int chunk, int NS, float *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t *full = (uint64_t *)(sm + (size_t)NS * chunk), *empty = full + NS;
  long nch = bytes / chunk;
  long c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
  int T = (int)(c1 - c0);
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) { for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) for (int t = 0; t < T; ++t) { int s = t % NS; mbar_wait(&empty[s], ((t / NS) & 1) ^ 1); expect_tx(&full[s], chunk); bulk(sm + (size_t)s * chunk, x + (c0 + t) * (long)chunk, chunk, &full[s]); }
  } else if (warp >= 2) {
    float a = 0;
    for (int t = 0; t < T; ++t) { int s = t % NS; mbar_wait(&full[s], (t / NS) & 1); a += ((float *)(sm + (size_t)s * chunk))[tid]; __syncwarp(); if (lane == 0) arrive(&empty[s]); }
    if (a == 12345.f) out[0] = a;
  }
}
extern "C" float run_ldg(const float *x, long bytes, float *out, int grid, int block, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_ldg<<<grid, block>>>((const float4 *)x, bytes / 16, out);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k_ldg<<<grid, block>>>((const float4 *)x, bytes / 16, out);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
extern "C" float run_bulk(const char *x, long bytes, float *out, int chunk, int NS, int grid, int reps) {
  size_t smem = (size_t)NS * chunk + 2 * NS * 8;
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_bulk<<<grid, 320, smem>>>(x, bytes, chunk, NS, out);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k_bulk<<<grid, 320, smem>>>(x, bytes, chunk, NS, out);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms / reps;
}
