// 1-D row partition of a (Cuthill-McKee ordered) matrix for the distributed
// solver: row ranges, halo plan for the SpMM, local CSR with columns remapped
// into [local rows | halo rows].  Every rank holds the full matrix (the setup
// is replicated), so each rank derives every peer's halo request locally --
// no planning collective is needed and all ranks agree by construction.
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "mg_block.cuh"
#include "mg_dist.cuh"

namespace mg {

std::vector<int64_t> row_ranges(int64_t n, int nranks) {
  std::vector<int64_t> rs(nranks + 1);
  for (int p = 0; p <= nranks; ++p) rs[p] = n * p / nranks;
  return rs;
}

void plan_from_halos(const std::vector<int64_t> &rs, int me,
                     const std::vector<std::vector<int64_t>> &halos, HostPlan &hp) {
  const int R = (int)rs.size() - 1;
  hp.rs = rs;
  hp.r0 = rs[me];
  hp.nloc = rs[me + 1] - rs[me];
  hp.halo = halos[me];
  hp.roff.assign(R, 0);
  hp.rcnt.assign(R, 0);
  for (int p = 0; p < R; ++p) {
    auto lo = std::lower_bound(hp.halo.begin(), hp.halo.end(), rs[p]);
    auto hi = std::lower_bound(hp.halo.begin(), hp.halo.end(), rs[p + 1]);
    hp.roff[p] = lo - hp.halo.begin();
    hp.rcnt[p] = hi - lo;
  }
  // to peer p: the rows of mine in p's halo, in p's (sorted) order, so they
  // land exactly in p's receive slots for me
  hp.soff.assign(R, 0);
  hp.scnt.assign(R, 0);
  hp.send_rows.clear();
  for (int p = 0; p < R; ++p) {
    hp.soff[p] = (int64_t)hp.send_rows.size();
    if (p == me) continue;
    for (int64_t j : halos[p])
      if (j >= hp.r0 && j < hp.r0 + hp.nloc) hp.send_rows.push_back((int)(j - hp.r0));
    hp.scnt[p] = (int64_t)hp.send_rows.size() - hp.soff[p];
  }
}

void host_plan(int64_t n, const int64_t *ptr, const int64_t *idx, int nranks, int me, HostPlan &hp,
               std::vector<int> *local_idx) {
  require(nranks >= 1 && me >= 0 && me < nranks, MG_ERR_INPUT, "bad rank / world size");
  auto rs = row_ranges(n, nranks);
  std::vector<std::vector<int64_t>> halos(nranks);
  for (int p = 0; p < nranks; ++p) {
    std::vector<int64_t> &h = halos[p];
    for (int64_t k = ptr[rs[p]]; k < ptr[rs[p + 1]]; ++k) {
      const int64_t j = idx[k];
      require(j >= 0 && j < n, MG_ERR_INPUT, "column index out of range");
      if (j < rs[p] || j >= rs[p + 1]) h.push_back(j);
    }
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
  }
  plan_from_halos(rs, me, halos, hp);
  if (local_idx) {
    local_idx->clear();
    for (int64_t k = ptr[hp.r0]; k < ptr[hp.r0 + hp.nloc]; ++k) {
      const int64_t j = idx[k];
      if (j >= hp.r0 && j < hp.r0 + hp.nloc)
        local_idx->push_back((int)(j - hp.r0));
      else
        local_idx->push_back(
            (int)(hp.nloc + (std::lower_bound(hp.halo.begin(), hp.halo.end(), j) - hp.halo.begin())));
    }
  }
}

// flag entries of rows [r0, r1) whose column is outside [r0, r1)
__global__ void k_remote_cols(int64_t base, int64_t cnt, int64_t r0, int64_t r1,
                              const int64_t *__restrict__ idx, int *__restrict__ out,
                              unsigned char *__restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx[base + e];
    out[e] = (int)j;
    flag[e] = (j < r0 || j >= r1) ? 1 : 0;
  }
}

// sorted unique remote columns of rows [r0, r1)
static void remote_unique(mg_ctx *ctx, const int64_t *ptr_h, const int64_t *idx, int64_t r0,
                          int64_t r1, DBuf<int> &out, int64_t &count) {
  const int64_t base = ptr_h[r0], cnt = ptr_h[r1] - ptr_h[r0];
  count = 0;
  out.alloc(ctx, 1);
  if (cnt == 0) return;
  DBuf<int> cols(ctx, cnt), sel(ctx, cnt), sorted(ctx, cnt);
  DBuf<unsigned char> flag(ctx, cnt);
  DBuf<int64_t> nsel(ctx, 1);
  k_remote_cols<<<grid_for(cnt, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
      base, cnt, r0, r1, idx, cols.p, flag.p);
  MG_CHECK_LAUNCH(ctx);
  size_t tb = 0;
  MG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cols.p, flag.p, sel.p, nsel.p, cnt,
                                     ctx->stream));
  DBuf<char> t(ctx, tb);
  MG_CUDA(cub::DeviceSelect::Flagged(t.p, tb, cols.p, flag.p, sel.p, nsel.p, cnt, ctx->stream));
  ctx->launches++;
  int64_t ns = 0;
  d2h_sync(ctx, &ns, nsel.p, sizeof(int64_t));
  if (ns == 0) return;
  size_t tb2 = 0;
  MG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, sel.p, sorted.p, (int)ns, 0, 32,
                                         ctx->stream));
  DBuf<char> t2(ctx, tb2);
  MG_CUDA(cub::DeviceRadixSort::SortKeys(t2.p, tb2, sel.p, sorted.p, (int)ns, 0, 32, ctx->stream));
  ctx->launches++;
  out.alloc(ctx, ns);
  size_t tb3 = 0;
  MG_CUDA(cub::DeviceSelect::Unique(nullptr, tb3, sorted.p, out.p, nsel.p, ns, ctx->stream));
  DBuf<char> t3(ctx, tb3);
  MG_CUDA(cub::DeviceSelect::Unique(t3.p, tb3, sorted.p, out.p, nsel.p, ns, ctx->stream));
  ctx->launches++;
  d2h_sync(ctx, &count, nsel.p, sizeof(int64_t));
}

template <typename T>
__global__ void k_local_csr(int64_t nloc, int64_t r0, const int64_t *__restrict__ ptr,
                            const int64_t *__restrict__ idx, const double *__restrict__ val,
                            const int *__restrict__ halo, int64_t nh, int64_t *__restrict__ lptr,
                            int *__restrict__ lidx, T *__restrict__ lval, T *__restrict__ rowsum) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gr = r0 + r, s = ptr[gr], e = ptr[gr + 1], o = s - ptr[r0];
    lptr[r] = o;
    if (r == nloc - 1) lptr[nloc] = e - ptr[r0];
    double rs = 0.0;
    for (int64_t k = s; k < e; ++k) {
      const int64_t j = idx[k];
      int lj;
      if (j >= r0 && j < r0 + nloc) {
        lj = (int)(j - r0);
      } else {
        int64_t lo = 0, hi = nh;  // lower_bound in the sorted halo list
        while (lo < hi) {
          int64_t mid = (lo + hi) >> 1;
          if (halo[mid] < j) lo = mid + 1;
          else hi = mid;
        }
        lj = (int)(nloc + lo);
      }
      lidx[o + (k - s)] = lj;
      lval[o + (k - s)] = (T)val[k];
      rs += val[k];
    }
    if (rowsum) rowsum[r] = (T)rs;
  }
}

__global__ void k_row_has_halo(int64_t nloc, const int64_t *__restrict__ lptr,
                               const int *__restrict__ lidx, int *__restrict__ flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc;
       r += (int64_t)gridDim.x * blockDim.x) {
    int f = 0;
    for (int64_t k = lptr[r]; k < lptr[r + 1]; ++k) f |= lidx[k] >= nloc;
    flag[r] = f;
  }
}

template <typename T>
void build_dist(mg_ctx *ctx, Comm *comm, int64_t n, const int64_t *ptr, const int64_t *idx,
                const double *val, DistPart<T> &dp) {
  const int R = comm->nranks, me = comm->rank;
  dp.rs = row_ranges(n, R);
  dp.r0 = dp.rs[me];
  dp.nloc = dp.rs[me + 1] - dp.rs[me];
  std::vector<int64_t> ptr_h(n + 1);
  d2h_sync(ctx, ptr_h.data(), ptr, (n + 1) * sizeof(int64_t));
  // sorted remote-column list of every rank (each derived locally: the
  // matrix is replicated), then the shared host planner
  std::vector<std::vector<int64_t>> halos(R);
  DBuf<int> mine;
  for (int p = 0; p < R; ++p) {
    DBuf<int> lst;
    int64_t cnt = 0;
    remote_unique(ctx, ptr_h.data(), idx, dp.rs[p], dp.rs[p + 1], lst, cnt);
    std::vector<int> h(cnt);
    if (cnt) d2h_sync(ctx, h.data(), lst.p, cnt * sizeof(int));
    halos[p].assign(h.begin(), h.end());
    if (p == me) {
      mine.alloc(ctx, cnt > 0 ? cnt : 1);
      if (cnt)
        MG_CUDA(cudaMemcpyAsync(mine.p, lst.p, cnt * sizeof(int), cudaMemcpyDeviceToDevice,
                                ctx->stream));
      sync(ctx);
    }
  }
  HostPlan hp;
  plan_from_halos(dp.rs, me, halos, hp);
  dp.nhalo = (int64_t)hp.halo.size();
  dp.roff = hp.roff;
  dp.rcnt = hp.rcnt;
  dp.soff = hp.soff;
  dp.scnt = hp.scnt;
  const std::vector<int> &send_h = hp.send_rows;
  dp.nsend = (int64_t)send_h.size();
  dp.send_rows.alloc(ctx, dp.nsend > 0 ? dp.nsend : 1);
  if (dp.nsend)
    MG_CUDA(cudaMemcpyAsync(dp.send_rows.p, send_h.data(), dp.nsend * sizeof(int),
                            cudaMemcpyHostToDevice, ctx->stream));
  // local CSR
  const int64_t lnnz = ptr_h[dp.r0 + dp.nloc] - ptr_h[dp.r0];
  dp.A.ptr.alloc(ctx, dp.nloc + 1);
  dp.A.idx.alloc(ctx, lnnz > 0 ? lnnz : 1);
  dp.A.val.alloc(ctx, lnnz > 0 ? lnnz : 1);
  const char *env = getenv("MG_SPMM_DIFF");
  const bool diff = sizeof(T) == 4 && !(env && env[0] == '0');
  if (diff) dp.A.rowsum.alloc(ctx, dp.nloc > 0 ? dp.nloc : 1);
  if (dp.nloc > 0) {
    k_local_csr<T><<<grid_for(dp.nloc, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        dp.nloc, dp.r0, ptr, idx, val, mine.p, dp.nhalo, dp.A.ptr.p, dp.A.idx.p, dp.A.val.p,
        diff ? dp.A.rowsum.p : nullptr);
    MG_CHECK_LAUNCH(ctx);
  }
  dp.A.view.n = dp.nloc;
  dp.A.view.nnz = lnnz;
  dp.A.view.ptr = dp.A.ptr.p;
  dp.A.view.idx = dp.A.idx.p;
  dp.A.view.val = dp.A.val.p;
  dp.A.view.rowsum = diff ? dp.A.rowsum.p : nullptr;
  // interior / boundary row lists (ascending local ids)
  std::vector<int> ri, rb;
  if (dp.nloc > 0) {
    DBuf<int> flag(ctx, dp.nloc);
    k_row_has_halo<<<grid_for(dp.nloc, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        dp.nloc, dp.A.ptr.p, dp.A.idx.p, flag.p);
    MG_CHECK_LAUNCH(ctx);
    std::vector<int> fh(dp.nloc);
    d2h_sync(ctx, fh.data(), flag.p, dp.nloc * sizeof(int));
    for (int64_t r = 0; r < dp.nloc; ++r) (fh[r] ? rb : ri).push_back((int)r);
  }
  dp.n_int = (int64_t)ri.size();
  dp.n_bnd = (int64_t)rb.size();
  dp.rows_int.alloc(ctx, std::max<int64_t>(dp.n_int, 1));
  dp.rows_bnd.alloc(ctx, std::max<int64_t>(dp.n_bnd, 1));
  if (dp.n_int)
    MG_CUDA(cudaMemcpyAsync(dp.rows_int.p, ri.data(), dp.n_int * sizeof(int),
                            cudaMemcpyHostToDevice, ctx->stream));
  if (dp.n_bnd)
    MG_CUDA(cudaMemcpyAsync(dp.rows_bnd.p, rb.data(), dp.n_bnd * sizeof(int),
                            cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);
}

template void build_dist<float>(mg_ctx *, Comm *, int64_t, const int64_t *, const int64_t *,
                                const double *, DistPart<float> &);
template void build_dist<double>(mg_ctx *, Comm *, int64_t, const int64_t *, const int64_t *,
                                 const double *, DistPart<double> &);

}  // namespace mg
