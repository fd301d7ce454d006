// Runtime plumbing: last-error storage, staging copies, scans.
#include <cub/device/device_scan.cuh>

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

void d2h_sync(mg_ctx *ctx, void *host, const void *dev, size_t bytes) {
  if (!bytes) return;
  ensure_pinned(ctx, bytes);
  MG_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(host, ctx->pinned, bytes);
}

void h2d(mg_ctx *ctx, void *dev, const void *host, size_t bytes) {
  if (!bytes) return;
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
