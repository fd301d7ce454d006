// NCCL (dlopen) and thread-local-rank implementations of mg::Comm.
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <mutex>

#include "mg_comm.cuh"

namespace mg {

// ------------------------------------------------------------------- NCCL ---
// Minimal NCCL ABI (nccl.h, NCCL 2.x): opaque comm, 128-byte unique id.
typedef void *ncclComm_t_;
typedef struct {
  char internal[128];
} ncclUniqueId_;
enum { kNcclUint8 = 1, kNcclDouble = 8 };
enum { kNcclSum = 0, kNcclMax = 2 };

struct NcclApi {
  void *h = nullptr;
  int (*GetUniqueId)(ncclUniqueId_ *);
  int (*CommInitRank)(ncclComm_t_ *, int, ncclUniqueId_, int);
  int (*CommDestroy)(ncclComm_t_);
  int (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t_, cudaStream_t);
  int (*Send)(const void *, size_t, int, int, ncclComm_t_, cudaStream_t);
  int (*Recv)(void *, size_t, int, int, ncclComm_t_, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  const char *(*GetErrorString)(int);
};

static NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.GetUniqueId = (int (*)(ncclUniqueId_ *))dlsym(api.h, "ncclGetUniqueId");
    api.CommInitRank = (int (*)(ncclComm_t_ *, int, ncclUniqueId_, int))dlsym(api.h, "ncclCommInitRank");
    api.CommDestroy = (int (*)(ncclComm_t_))dlsym(api.h, "ncclCommDestroy");
    api.AllReduce = (int (*)(const void *, void *, size_t, int, int, ncclComm_t_, cudaStream_t))dlsym(
        api.h, "ncclAllReduce");
    api.Send = (int (*)(const void *, size_t, int, int, ncclComm_t_, cudaStream_t))dlsym(api.h, "ncclSend");
    api.Recv = (int (*)(void *, size_t, int, int, ncclComm_t_, cudaStream_t))dlsym(api.h, "ncclRecv");
    api.GroupStart = (int (*)())dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (int (*)())dlsym(api.h, "ncclGroupEnd");
    api.GetErrorString = (const char *(*)(int))dlsym(api.h, "ncclGetErrorString");
  });
  require(api.h != nullptr && api.AllReduce != nullptr, MG_ERR_NCCL,
          "libnccl.so.2 not found (import torch first, or add nvidia/nccl/lib to the loader path)");
  return api;
}

#define MG_NCCL(expr)                                                                     \
  do {                                                                                    \
    int _r = (expr);                                                                      \
    if (_r != 0)                                                                          \
      throw Error(MG_ERR_NCCL, std::string(#expr) + ": " +                                \
                                   (nccl().GetErrorString ? nccl().GetErrorString(_r) : "?")); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t_ comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allreduce(mg_ctx *ctx, double *buf, size_t count, bool max_op) override {
    if (nranks == 1 || count == 0) return;
    MG_NCCL(nccl().AllReduce(buf, buf, count, kNcclDouble, max_op ? kNcclMax : kNcclSum, comm,
                             ctx->stream));
  }
  void exchange(mg_ctx *ctx, const void *sendbuf, const int64_t *soff, const int64_t *scnt,
                void *recvbuf, const int64_t *roff, const int64_t *rcnt, size_t elem) override {
    if (nranks == 1) return;
    MG_NCCL(nccl().GroupStart());
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      if (scnt[p])
        MG_NCCL(nccl().Send((const char *)sendbuf + soff[p] * elem, scnt[p] * elem, kNcclUint8, p,
                            comm, ctx->stream));
      if (rcnt[p])
        MG_NCCL(nccl().Recv((char *)recvbuf + roff[p] * elem, rcnt[p] * elem, kNcclUint8, p, comm,
                            ctx->stream));
    }
    MG_NCCL(nccl().GroupEnd());
  }
};

void nccl_unique_id(void *out128) {
  ncclUniqueId_ id;
  MG_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
}

Comm *make_nccl_comm(int nranks, int rank, const void *uid) {
  auto *c = new NcclComm();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId_ id;
  std::memcpy(&id, uid, sizeof(id));
  int r = nccl().CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    delete c;
    throw Error(MG_ERR_NCCL, std::string("ncclCommInitRank: ") +
                                 (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
  }
  return c;
}

// -------------------------------------------------------------- LocalComm ---
struct LocalGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<std::vector<double>> host;                 // allreduce slots
  std::vector<const void *> sbuf;
  std::vector<const int64_t *> soff, scnt;
  explicit LocalGroup(int n_) : n(n_), host(n_), sbuf(n_), soff(n_), scnt(n_) {}
  // a rank that failed alone never arrives: time out instead of hanging
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; })) {
      throw Error(MG_ERR_INTERNAL, "local communicator: peer rank did not arrive (120 s)");
    }
  }
};

struct LocalComm : Comm {
  LocalGroup *g;
  void allreduce(mg_ctx *ctx, double *buf, size_t count, bool max_op) override {
    if (nranks == 1 || count == 0) return;
    g->host[rank].resize(count);
    MG_CUDA(cudaMemcpyAsync(g->host[rank].data(), buf, count * sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
    g->barrier();
    std::vector<double> acc(g->host[0]);
    for (int p = 1; p < nranks; ++p)
      for (size_t i = 0; i < count; ++i)
        acc[i] = max_op ? std::max(acc[i], g->host[p][i]) : acc[i] + g->host[p][i];
    g->barrier();  // every rank has read every slot
    MG_CUDA(cudaMemcpyAsync(buf, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  void exchange(mg_ctx *ctx, const void *sendbuf, const int64_t *soff, const int64_t *scnt,
                void *recvbuf, const int64_t *roff, const int64_t *rcnt, size_t elem) override {
    if (nranks == 1) return;
    MG_CUDA(cudaStreamSynchronize(ctx->stream));  // send buffers are packed
    g->sbuf[rank] = sendbuf;
    g->soff[rank] = soff;
    g->scnt[rank] = scnt;
    g->barrier();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank || !rcnt[p]) continue;
      require(g->scnt[p][rank] == rcnt[p], MG_ERR_INTERNAL, "halo plan mismatch between ranks");
      MG_CUDA(cudaMemcpyAsync((char *)recvbuf + roff[p] * elem,
                              (const char *)g->sbuf[p] + g->soff[p][rank] * elem, rcnt[p] * elem,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    }
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
    g->barrier();  // peers may reuse their send buffers
  }
};

void *local_comm_group_create(int nranks) { return new LocalGroup(nranks); }
void local_comm_group_destroy(void *group) { delete (LocalGroup *)group; }
Comm *local_comm_rank(void *group, int rank) {
  auto *c = new LocalComm();
  c->g = (LocalGroup *)group;
  c->nranks = c->g->n;
  c->rank = rank;
  return c;
}

}  // namespace mg
