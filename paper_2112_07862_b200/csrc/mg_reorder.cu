// Locality ordering of the graph for the solver (Cuthill-McKee by levels).
//
// The kNN graphs of the configs arrive in random node order, so every SpMM
// gather W[j, :] of a neighbour row is a random HBM access and the working
// set of W (20M x 36 fp32 = 2.9 GB at config 5) cannot live in L2.  A
// breadth-first Cuthill-McKee numbering keeps every row's neighbours within
// roughly two BFS levels (a band of ~N^(2/3) rows on 3-D geometric graphs),
// so the gathered rows stay L2-resident.  The ordering is a pure relabeling:
// structure is preserved and all results are mapped back to the caller's
// node ids.  Deterministic: each level is sorted by (parent's new id, id).
#include <climits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "mg_graph.cuh"

namespace mg {

__global__ void k_cm_init(int64_t n, int *lev, unsigned long long *key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    lev[i] = -1;
    key[i] = ~0ull;
  }
}

// expand frontier F (in new-id order) by one level: claim unvisited
// neighbours, record the smallest parent new id per claimed node
__global__ void k_cm_expand(const int *__restrict__ F, int f, int64_t base_id,
                            const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                            int *lev, int L, unsigned long long *key, int *next, int *nnext) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
    const int u = F[t];
    const unsigned long long pid = (unsigned long long)(base_id + t);
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
      const int v = (int)idx[e];
      int lv = lev[v];
      if (lv == -1) {
        int old = atomicCAS(lev + v, -1, L + 1);
        if (old == -1) {
          next[atomicAdd(nnext, 1)] = v;
          lv = L + 1;
        } else {
          lv = old;
        }
      }
      if (lv == L + 1) atomicMin(key + v, pid);
    }
  }
}

__global__ void k_cm_keys(const int *__restrict__ next, int f, const unsigned long long *key,
                          unsigned long long *ck) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
    const int v = next[t];
    ck[t] = (key[v] << 32) | (unsigned long long)(unsigned)v;
  }
}

__global__ void k_cm_assign(const unsigned long long *__restrict__ ck, int f, int64_t base,
                            int *F, int64_t *perm, int64_t *inv) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
    const int v = (int)(ck[t] & 0xffffffffull);
    F[t] = v;
    perm[base + t] = v;
    inv[v] = base + t;
  }
}

__global__ void k_cm_seed(int v, int64_t base, int *lev, int L, int *F, int64_t *perm,
                          int64_t *inv) {
  lev[v] = L;
  F[0] = v;
  perm[base] = v;
  inv[v] = base;
}

// first unvisited node (components are visited in increasing smallest id)
__global__ void k_cm_first_unvisited(const int *lev, int64_t n, int64_t from, int *out) {
  for (int64_t i = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (lev[i] == -1) atomicMin(out, (int)i);
}

void cm_order(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, int64_t *perm,
              int64_t *inv) {
  require(n < INT_MAX, MG_ERR_INPUT, "graph too large for 32-bit node ids");
  DBuf<int> lev(ctx, n), F(ctx, n), next(ctx, n), cnt(ctx, 2);
  DBuf<unsigned long long> key(ctx, n), ck(ctx, n), ck2(ctx, n);
  const int g = grid_for(n, 256, ctx->num_sms * 16);
  k_cm_init<<<g, 256, 0, ctx->stream>>>(n, lev.p, key.p);
  MG_CHECK_LAUNCH(ctx);
  size_t tmp_bytes = 0;
  MG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, ck.p, ck2.p, (int)n, 0, 64,
                                         ctx->stream));
  DBuf<char> tmp(ctx, tmp_bytes);
  int64_t assigned = 0, from = 0;
  int L = 0;
  while (assigned < n) {
    // seed of the next component: smallest unvisited id
    int seed = INT_MAX;
    MG_CUDA(cudaMemcpyAsync(cnt.p, &seed, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    k_cm_first_unvisited<<<grid_for(n - from, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        lev.p, n, from, cnt.p);
    MG_CHECK_LAUNCH(ctx);
    d2h_sync(ctx, &seed, cnt.p, sizeof(int));
    if (seed == INT_MAX) break;
    from = seed;
    k_cm_seed<<<1, 1, 0, ctx->stream>>>(seed, assigned, lev.p, L, F.p, perm, inv);
    MG_CHECK_LAUNCH(ctx);
    int64_t fbase = assigned;  // new id of F[0]
    int f = 1;
    assigned += 1;
    while (f > 0) {
      MG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), ctx->stream));
      k_cm_expand<<<grid_for(f, 128, ctx->num_sms * 16), 128, 0, ctx->stream>>>(
          F.p, f, fbase, ptr, idx, lev.p, L, key.p, next.p, cnt.p);
      MG_CHECK_LAUNCH(ctx);
      int nf = 0;
      d2h_sync(ctx, &nf, cnt.p, sizeof(int));
      ++L;
      if (nf == 0) break;
      k_cm_keys<<<grid_for(nf, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(next.p, nf, key.p,
                                                                            ck.p);
      MG_CHECK_LAUNCH(ctx);
      MG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, ck.p, ck2.p, nf, 0, 64,
                                             ctx->stream));
      ctx->launches++;
      k_cm_assign<<<grid_for(nf, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          ck2.p, nf, assigned, F.p, perm, inv);
      MG_CHECK_LAUNCH(ctx);
      fbase = assigned;
      assigned += nf;
      f = nf;
    }
    ++L;
  }
  require(assigned == n, MG_ERR_INTERNAL, "ordering did not visit every node");
}

// ---- symmetric permutation of a CSR graph: new row r = old row perm[r] ----
__global__ void k_perm_rowlen(int64_t n, const int64_t *__restrict__ ptr,
                              const int64_t *__restrict__ perm, int64_t *len) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = perm[r];
    len[r] = ptr[o + 1] - ptr[o];
  }
}

__global__ void k_perm_gather(int64_t n, const int64_t *__restrict__ ptr,
                              const int64_t *__restrict__ idx, const double *__restrict__ w,
                              const int64_t *__restrict__ perm, const int64_t *__restrict__ inv,
                              const int64_t *__restrict__ nptr, int64_t *nidx, double *nw) {
  // one warp per new row
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t o = perm[r];
    const int64_t s = ptr[o], e = ptr[o + 1], d = nptr[r];
    for (int64_t k = s + lane; k < e; k += 32) {
      nidx[d + (k - s)] = inv[idx[k]];
      nw[d + (k - s)] = w[k];
    }
  }
}

void permute_graph(mg_ctx *ctx, int64_t n, const int64_t *ptr, const int64_t *idx, const double *w,
                   const int64_t *perm, const int64_t *inv, int64_t *nptr, int64_t *nidx,
                   double *nw) {
  DBuf<int64_t> len(ctx, n + 1);
  MG_CUDA(cudaMemsetAsync(len.p + n, 0, sizeof(int64_t), ctx->stream));
  k_perm_rowlen<<<grid_for(n, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(n, ptr, perm,
                                                                              len.p);
  MG_CHECK_LAUNCH(ctx);
  const int64_t nnz = exclusive_scan_i64(ctx, len.p, nptr, n);
  if (nnz == 0) return;
  DBuf<int64_t> tidx(ctx, nnz);
  DBuf<double> tw(ctx, nnz);
  k_perm_gather<<<grid_for(n * 32, 256, ctx->num_sms * 32), 256, 0, ctx->stream>>>(
      n, ptr, idx, w, perm, inv, nptr, tidx.p, tw.p);
  MG_CHECK_LAUNCH(ctx);
  // sort each row by its new column ids (rows are short; segmented sort)
  size_t tb = 0;
  MG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, tidx.p, nidx, tw.p, nw, nnz, n, nptr,
                                              nptr + 1, ctx->stream));
  DBuf<char> t(ctx, tb);
  MG_CUDA(cub::DeviceSegmentedSort::SortPairs(t.p, tb, tidx.p, nidx, tw.p, nw, nnz, n, nptr,
                                              nptr + 1, ctx->stream));
  ctx->launches++;
}

}  // namespace mg
