// Collectives for the 1-D row-partitioned solver.
//
//   NcclComm  - one process per GPU; NCCL (libnccl.so.2, loaded with dlopen so
//               the library has no link-time NCCL dependency) over NVLink /
//               NVSwitch: allreduce of the small Gram / norm blocks, grouped
//               send/recv for the SpMM halo rows.
//   LocalComm - R virtual ranks as host threads of one process sharing one
//               GPU (each with its own context/stream); collectives via host
//               rendezvous + device copies.  Used to test the partitioned
//               algorithm end-to-end on a single B200 (no kernel ever waits
//               on another rank's kernel).
#pragma once
#include "mg_common.cuh"

namespace mg {

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // in-place sum / max over ranks of a device fp64 array (stream-ordered on ctx)
  virtual void allreduce(mg_ctx *ctx, double *buf, size_t count, bool max_op) = 0;
  // point-to-point exchange: to peer p send scnt[p] elements from sendbuf+soff[p],
  // receive rcnt[p] elements into recvbuf+roff[p]; elem = element size in bytes
  virtual void exchange(mg_ctx *ctx, const void *sendbuf, const int64_t *soff,
                        const int64_t *scnt, void *recvbuf, const int64_t *roff,
                        const int64_t *rcnt, size_t elem) = 0;
};

Comm *make_nccl_comm(int nranks, int rank, const void *unique_id128);
void nccl_unique_id(void *out128);
Comm *local_comm_rank(void *group, int rank);
void *local_comm_group_create(int nranks);
void local_comm_group_destroy(void *group);

}  // namespace mg

struct mg_comm {
  mg::Comm *impl = nullptr;
};
