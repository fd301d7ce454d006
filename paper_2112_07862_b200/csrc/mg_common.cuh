// Common plumbing for the manigraph B200 native library: context, status
// handling, stream-ordered workspace, launch accounting, warp helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/manigraph_b200.h"

namespace mg {

// ---------------------------------------------------------------- errors ---
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);

#define MG_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw ::mg::Error(MG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                         " @" __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

#define MG_CHECK_LAUNCH(ctx)                                                       \
  do {                                                                             \
    (ctx)->launches++;                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      throw ::mg::Error(MG_ERR_CUDA, std::string("kernel launch: ") +              \
                                         cudaGetErrorString(_e) + " @" __FILE__ ":" + \
                                         std::to_string(__LINE__));                \
  } while (0)

inline void require(bool ok, int code, const std::string &msg) {
  if (!ok) throw Error(code, msg);
}

}  // namespace mg

// ---------------------------------------------------------------- context ---
struct mg_prof_rec {
  int cls;                 // kernel class (mg_prof_class)
  double bytes;            // algorithmic bytes of this launch
  cudaEvent_t start, stop;
};

struct mg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  void *pinned = nullptr;       // small pinned staging buffer for D2H scalars
  size_t pinned_bytes = 0;
  void *stage[2] = {nullptr, nullptr};  // pinned ring for large host <-> device copies
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int profiling = 0;            // record CUDA events around hot kernels
  std::vector<mg_prof_rec> prof;
  std::vector<cudaEvent_t> event_pool;
};

namespace mg {

// Stream-ordered device buffer (cudaMallocAsync on the context stream).
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(mg_ctx *ctx, size_t count) { alloc(ctx, count); }
  void alloc(mg_ctx *ctx, size_t count) {
    release();
    s = ctx->stream;
    n = count;
    if (count) {
      cudaError_t e = cudaMallocAsync((void **)&p, count * sizeof(T), s);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(MG_ERR_NOMEM, "cudaMallocAsync of " + std::to_string(count * sizeof(T)) +
                                      " bytes failed: " + cudaGetErrorString(e));
      }
    }
  }
  void zero() {
    if (n) MG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  T *get() const { return p; }
  operator T *() const { return p; }
};

// Hot-kernel timing (enabled by mg_ctx_set_profiling): events on ctx->stream.
enum ProfClass { PROF_SPMM = 0, PROF_GRAM = 1, PROF_UPDATE = 2, PROF_RESID = 3, PROF_CTRL = 4,
                 PROF_SETUP = 5, PROF_NCLASS = 6 };
struct ProfScope {
  mg_ctx *ctx;
  int idx = -1;
  ProfScope(mg_ctx *c, int cls, double bytes);
  ~ProfScope();
};

// Large host <-> device copies (pageable host memory): pipelined through two
// pinned 64 MB stages, the host-side memcpy split over threads.
void d2h_large(mg_ctx *ctx, void *host, const void *dev, size_t bytes);
void h2d_large(mg_ctx *ctx, void *dev, const void *host, size_t bytes);
void free_stages(mg_ctx *ctx);

// Copy device -> host through the context's pinned staging area and wait.
void d2h_sync(mg_ctx *ctx, void *host, const void *dev, size_t bytes);
void h2d(mg_ctx *ctx, void *dev, const void *host, size_t bytes);  // synchronous w.r.t. host buffer
void sync(mg_ctx *ctx);

inline int grid_for(int64_t work, int block, int cap) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// exclusive scan of int64 counts (n entries) into out (n+1 entries), returns total
int64_t exclusive_scan_i64(mg_ctx *ctx, const int64_t *counts, int64_t *out, int64_t n);

// ------------------------------------------------------------ warp helpers ---
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace mg
