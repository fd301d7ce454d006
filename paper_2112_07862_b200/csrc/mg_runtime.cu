// Runtime plumbing: last-error storage, staging copies, scans.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <thread>
#include <vector>

#include "mg_common.cuh"

namespace mg {

static thread_local std::string g_last_error;

void set_last_error(const std::string &msg) { g_last_error = msg; }
const char *last_error_cstr() { return g_last_error.c_str(); }

static void ensure_pinned(mg_ctx *ctx, size_t bytes) {
  if (ctx->pinned_bytes >= bytes) return;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  size_t cap = bytes < 65536 ? 65536 : bytes;
  MG_CUDA(cudaMallocHost(&ctx->pinned, cap));
  ctx->pinned_bytes = cap;
}

static constexpr size_t kStageBytes = 64ull << 20;

static void ensure_stages(mg_ctx *ctx) {
  for (int i = 0; i < 2; ++i)
    if (!ctx->stage[i]) {
      MG_CUDA(cudaMallocHost(&ctx->stage[i], kStageBytes));
      MG_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
    }
}

void free_stages(mg_ctx *ctx) {
  for (int i = 0; i < 2; ++i) {
    if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
    if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
    ctx->stage[i] = nullptr;
    ctx->stage_ev[i] = nullptr;
  }
}

static void par_memcpy(void *dst, const void *src, size_t bytes) {
  const int hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::min<size_t>(std::min(hw, 16), bytes / (4u << 20) + 1);
  if (T <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const size_t a = bytes * t / T, b = bytes * (t + 1) / T;
    th.emplace_back([=]() {
      std::memcpy((char *)dst + a, (const char *)src + a, b - a);
    });
  }
  for (auto &x : th) x.join();
}

void d2h_large(mg_ctx *ctx, void *host, const void *dev, size_t bytes) {
  if (!bytes) return;
  ensure_stages(ctx);
  const size_t nch = (bytes + kStageBytes - 1) / kStageBytes;
  for (size_t c = 0; c <= nch; ++c) {
    if (c < nch) {  // DMA chunk c into stage c % 2
      const size_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
      MG_CUDA(cudaMemcpyAsync(ctx->stage[c & 1], (const char *)dev + off, len,
                              cudaMemcpyDeviceToHost, ctx->stream));
      MG_CUDA(cudaEventRecord(ctx->stage_ev[c & 1], ctx->stream));
    }
    if (c > 0) {  // drain chunk c - 1 while chunk c is in flight
      const size_t p = c - 1, off = p * kStageBytes, len = std::min(kStageBytes, bytes - off);
      MG_CUDA(cudaEventSynchronize(ctx->stage_ev[p & 1]));
      par_memcpy((char *)host + off, ctx->stage[p & 1], len);
    }
  }
}

void h2d_large(mg_ctx *ctx, void *dev, const void *host, size_t bytes) {
  if (!bytes) return;
  ensure_stages(ctx);
  const size_t nch = (bytes + kStageBytes - 1) / kStageBytes;
  for (size_t c = 0; c < nch; ++c) {
    const size_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
    if (c >= 2) MG_CUDA(cudaEventSynchronize(ctx->stage_ev[c & 1]));  // stage free again
    par_memcpy(ctx->stage[c & 1], (const char *)host + off, len);
    MG_CUDA(cudaMemcpyAsync((char *)dev + off, ctx->stage[c & 1], len, cudaMemcpyHostToDevice,
                            ctx->stream));
    MG_CUDA(cudaEventRecord(ctx->stage_ev[c & 1], ctx->stream));
  }
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void d2h_sync(mg_ctx *ctx, void *host, const void *dev, size_t bytes) {
  if (!bytes) return;
  if (bytes > (8u << 20)) {
    d2h_large(ctx, host, dev, bytes);
    return;
  }
  ensure_pinned(ctx, bytes);
  MG_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(host, ctx->pinned, bytes);
}

void h2d(mg_ctx *ctx, void *dev, const void *host, size_t bytes) {
  if (!bytes) return;
  if (bytes > (8u << 20)) {
    h2d_large(ctx, dev, host, bytes);
    return;
  }
  // small parameter blocks: stage through pinned memory; the copy must finish
  // before the staging area is reused, so wait for it.
  ensure_pinned(ctx, bytes);
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(ctx->pinned, host, bytes);
  MG_CUDA(cudaMemcpyAsync(dev, ctx->pinned, bytes, cudaMemcpyHostToDevice, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void sync(mg_ctx *ctx) { MG_CUDA(cudaStreamSynchronize(ctx->stream)); }

static cudaEvent_t take_event(mg_ctx *ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  MG_CUDA(cudaEventCreate(&e));
  return e;
}

ProfScope::ProfScope(mg_ctx *c, int cls, double bytes) : ctx(c) {
  if (!ctx->profiling) return;
  mg_prof_rec r;
  r.cls = cls;
  r.bytes = bytes;
  r.start = take_event(ctx);
  r.stop = take_event(ctx);
  MG_CUDA(cudaEventRecord(r.start, ctx->stream));
  idx = (int)ctx->prof.size();
  ctx->prof.push_back(r);
}

ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(ctx->prof[idx].stop, ctx->stream);
}

int64_t exclusive_scan_i64(mg_ctx *ctx, const int64_t *counts, int64_t *out, int64_t n) {
  // out has n+1 entries; out[n] = total
  size_t tmp = 0;
  MG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, out, n + 1, ctx->stream));
  DBuf<char> t(ctx, tmp);
  // counts must have n+1 readable entries with counts[n] == 0: callers allocate so.
  MG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, counts, out, n + 1, ctx->stream));
  ctx->launches++;
  int64_t total = 0;
  d2h_sync(ctx, &total, out + n, sizeof(int64_t));
  return total;
}

}  // namespace mg
