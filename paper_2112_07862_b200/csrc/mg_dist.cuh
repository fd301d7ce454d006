// Row-partition data of the distributed solver (mg_dist.cu).
#pragma once
#include "mg_block.cuh"
#include "mg_comm.cuh"

namespace mg {

// equal row ranges over the (locality-ordered) rows: rs[p] .. rs[p+1]
std::vector<int64_t> row_ranges(int64_t n, int nranks);

template <typename T>
struct DistPart {
  std::vector<int64_t> rs;        // row ranges (nranks + 1)
  int64_t r0 = 0, nloc = 0;       // my global row offset and count
  int64_t nhalo = 0;              // remote rows my SpMM reads (sorted by global id)
  std::vector<int64_t> roff, rcnt;  // per peer: halo rows received (offset/count, rows)
  std::vector<int64_t> soff, scnt;  // per peer: my rows sent (offset/count into send_rows)
  int64_t nsend = 0;
  DBuf<int> send_rows;            // local row ids to pack, grouped by peer
  OwnedCSR<T> A;                  // local rows, columns in [local | halo] numbering
  // local rows whose SpMM reads no halo row (interior) / some halo row
  // (boundary): the interior rows are formed while the halo exchange runs
  DBuf<int> rows_int, rows_bnd;
  int64_t n_int = 0, n_bnd = 0;
};

// halo plan from the sorted remote-column lists of every rank (host): the
// same function backs the device build and mg_dist_plan_host
struct HostPlan {
  int64_t r0 = 0, nloc = 0;
  std::vector<int64_t> rs, halo, roff, rcnt, soff, scnt;
  std::vector<int> send_rows;  // local row ids, grouped by peer
};
void plan_from_halos(const std::vector<int64_t> &rs, int me,
                     const std::vector<std::vector<int64_t>> &halos, HostPlan &hp);
// fully host-side plan (small graphs / tests): remote lists by a host scan
void host_plan(int64_t n, const int64_t *ptr, const int64_t *idx, int nranks, int me, HostPlan &hp,
               std::vector<int> *local_idx);

template <typename T>
void build_dist(mg_ctx *ctx, Comm *comm, int64_t n, const int64_t *ptr, const int64_t *idx,
                const double *val, DistPart<T> &dp);

}  // namespace mg
