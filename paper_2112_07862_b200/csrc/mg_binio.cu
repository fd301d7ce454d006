// Binary embedding / graph files: the same objects as the
// reference's text formats (embedding.py:131-166, graph.py:147-194) without
// the 17-digit text round trip.  The CSV of a 20M x 32 embedding is ~12 GB of
// text; here the arrays are written as they are in memory, by several
// threads at disjoint offsets (pwrite / pread).
//
// Layout (little-endian, 64-byte header, arrays 8-byte aligned):
//   embedding  "MGBEMB01" | u32 version=1 | u32 flags (1: b present) | i64 n |
//              i64 k | char method[16] | pad -> 64 |
//              f64 eigenvalues[k] | f64 P[n*k] (row-major) | f64 b[n] (flag 1)
//   graph      "MGBGRF01" | u32 version=1 | u32 0 | i64 n | i64 nnz | pad -> 64 |
//              i64 indptr[n+1] | i64 indices[nnz] | f64 weights[nnz]
// (canonical CSR of graph.py:20-29: both half-edges, rows ascending, no
// self-loops, w > 0 -- checked on load, errors as Graph.from_edges raises them)
#include <fcntl.h>
#include <unistd.h>

#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mg_common.cuh"

namespace mg {

namespace {

struct FileGuard {
  int fd = -1;
  ~FileGuard() {
    if (fd >= 0) close(fd);
  }
};

int nthreads(int t) {
  if (t > 0) return t;
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 16u));
}

// parallel pwrite / pread of one contiguous array at byte offset `off`
void par_io(int fd, bool wr, void *buf, size_t bytes, off_t off, int threads, const char *path) {
  if (!bytes) return;
  const size_t chunk = std::max<size_t>(size_t(8) << 20, (bytes + threads - 1) / threads);
  std::vector<std::thread> th;
  std::vector<int> err((bytes + chunk - 1) / chunk, 0);
  for (size_t c = 0, i = 0; c < bytes; c += chunk, ++i) {
    th.emplace_back([&, c, i] {
      size_t done = 0, len = std::min(chunk, bytes - c);
      char *p = static_cast<char *>(buf) + c;
      while (done < len) {
        const ssize_t r = wr ? pwrite(fd, p + done, len - done, off + (off_t)(c + done))
                             : pread(fd, p + done, len - done, off + (off_t)(c + done));
        if (r <= 0) {
          err[i] = r == 0 ? -1 : errno;
          return;
        }
        done += (size_t)r;
      }
    });
  }
  for (auto &t : th) t.join();
  for (int e : err)
    if (e) throw Error(MG_ERR_INPUT, std::string(path) + ": " + (e < 0 ? "truncated file" : strerror(e)));
}

int open_or_throw(const char *path, bool wr) {
  const int fd = wr ? open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644) : open(path, O_RDONLY);
  if (fd < 0) throw Error(MG_ERR_INPUT, std::string(path) + ": " + strerror(errno));
  return fd;
}

struct Header {
  char magic[8];
  uint32_t version, flags;
  int64_t a, b;
  char method[16];
  char pad[16];
};
static_assert(sizeof(Header) == 64, "header is 64 bytes");

Header read_header(int fd, const char *path, const char *magic) {
  Header h;
  if (pread(fd, &h, sizeof(h), 0) != (ssize_t)sizeof(h) || std::memcmp(h.magic, magic, 8) != 0)
    throw Error(MG_ERR_PARSE, std::string(path) + ": not a " + std::string(magic, 8) + " file");
  if (h.version != 1)
    throw Error(MG_ERR_PARSE, std::string(path) + ": unsupported version " + std::to_string(h.version));
  return h;
}

}  // namespace

void save_embedding_bin(const char *path, int64_t n, int64_t k, const double *P,
                        const double *eig, const double *b, const char *method, int threads) {
  require(n >= 0 && k >= 0, MG_ERR_INPUT, "embedding dimensions must be non-negative");
  FileGuard f;
  f.fd = open_or_throw(path, true);
  Header h{};
  std::memcpy(h.magic, "MGBEMB01", 8);
  h.version = 1;
  h.flags = b ? 1u : 0u;
  h.a = n;
  h.b = k;
  if (method) std::strncpy(h.method, method, sizeof(h.method) - 1);
  const int t = nthreads(threads);
  std::vector<double> ev(k, NAN);
  if (eig) std::memcpy(ev.data(), eig, k * sizeof(double));
  par_io(f.fd, true, &h, sizeof(h), 0, 1, path);
  off_t off = sizeof(h);
  par_io(f.fd, true, ev.data(), k * sizeof(double), off, 1, path);
  off += (off_t)(k * sizeof(double));
  par_io(f.fd, true, const_cast<double *>(P), (size_t)n * k * sizeof(double), off, t, path);
  off += (off_t)((size_t)n * k * sizeof(double));
  if (b) par_io(f.fd, true, const_cast<double *>(b), n * sizeof(double), off, t, path);
}

// P == nullptr: header only
void load_embedding_bin(const char *path, int64_t *n, int64_t *k, int *has_b, char *method,
                        double *P, double *eig, double *b, int threads) {
  FileGuard f;
  f.fd = open_or_throw(path, false);
  Header h = read_header(f.fd, path, "MGBEMB01");
  require(h.a >= 0 && h.b >= 0, MG_ERR_PARSE, std::string(path) + ": bad dimensions");
  *n = h.a;
  *k = h.b;
  *has_b = (h.flags & 1u) ? 1 : 0;
  if (method) {
    std::memcpy(method, h.method, 16);
    method[15] = 0;
  }
  if (!P) return;
  const int t = nthreads(threads);
  off_t off = sizeof(h);
  std::vector<double> ev(h.b);
  par_io(f.fd, false, ev.data(), h.b * sizeof(double), off, 1, path);
  if (eig) std::memcpy(eig, ev.data(), h.b * sizeof(double));
  off += (off_t)(h.b * sizeof(double));
  par_io(f.fd, false, P, (size_t)h.a * h.b * sizeof(double), off, t, path);
  off += (off_t)((size_t)h.a * h.b * sizeof(double));
  if (b && (h.flags & 1u)) par_io(f.fd, false, b, h.a * sizeof(double), off, t, path);
}

void save_graph_bin(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *w, int threads) {
  require(n >= 0, MG_ERR_INPUT, "n must be non-negative");
  const int64_t nnz = indptr[n];
  FileGuard f;
  f.fd = open_or_throw(path, true);
  Header h{};
  std::memcpy(h.magic, "MGBGRF01", 8);
  h.version = 1;
  h.a = n;
  h.b = nnz;
  const int t = nthreads(threads);
  par_io(f.fd, true, &h, sizeof(h), 0, 1, path);
  off_t off = sizeof(h);
  par_io(f.fd, true, const_cast<int64_t *>(indptr), (n + 1) * sizeof(int64_t), off, t, path);
  off += (off_t)((n + 1) * sizeof(int64_t));
  par_io(f.fd, true, const_cast<int64_t *>(indices), nnz * sizeof(int64_t), off, t, path);
  off += (off_t)(nnz * sizeof(int64_t));
  par_io(f.fd, true, const_cast<double *>(w), nnz * sizeof(double), off, t, path);
}

// indptr == nullptr: header only.  The CSR is validated as Graph.from_edges
// would have built it (graph.py:31-79): canonical rows, symmetric, w > 0.
void load_graph_bin(const char *path, int64_t *n, int64_t *nnz, int64_t *indptr, int64_t *indices,
                    double *w, int threads) {
  FileGuard f;
  f.fd = open_or_throw(path, false);
  Header h = read_header(f.fd, path, "MGBGRF01");
  require(h.a >= 0 && h.b >= 0, MG_ERR_PARSE, std::string(path) + ": bad dimensions");
  *n = h.a;
  *nnz = h.b;
  if (!indptr) return;
  const int t = nthreads(threads);
  off_t off = sizeof(h);
  par_io(f.fd, false, indptr, (h.a + 1) * sizeof(int64_t), off, t, path);
  off += (off_t)((h.a + 1) * sizeof(int64_t));
  par_io(f.fd, false, indices, h.b * sizeof(int64_t), off, t, path);
  off += (off_t)(h.b * sizeof(int64_t));
  par_io(f.fd, false, w, h.b * sizeof(double), off, t, path);
  const int64_t N = h.a;
  require(indptr[0] == 0 && indptr[N] == h.b, MG_ERR_PARSE, std::string(path) + ": bad indptr");
  // per-row checks in parallel; the first offending row wins
  std::vector<std::thread> th;
  std::vector<int64_t> bad(t, INT64_MAX);
  std::vector<std::string> why(t);
  for (int q = 0; q < t; ++q)
    th.emplace_back([&, q] {
      for (int64_t i = N * q / t; i < N * (q + 1) / t; ++i) {
        const int64_t s = indptr[i], e = indptr[i + 1];
        if (e < s || s < 0 || e > h.b) {
          bad[q] = i, why[q] = "bad indptr at row " + std::to_string(i);
          return;
        }
        for (int64_t p = s; p < e; ++p) {
          const int64_t j = indices[p];
          std::string m;
          if (j < 0 || j >= N) m = "edge references node " + std::to_string(j) + " >= n=" + std::to_string(N);
          else if (j == i) m = "self-loop on node " + std::to_string(i);
          else if (p > s && j <= indices[p - 1]) m = "row " + std::to_string(i) + " not strictly ascending";
          else if (!(w[p] > 0.0) || !std::isfinite(w[p]))
            m = "edge (" + std::to_string(std::min(i, j)) + ", " + std::to_string(std::max(i, j)) +
                ") has non-positive weight";
          if (!m.empty()) {
            bad[q] = i, why[q] = m;
            return;
          }
          // symmetric half-edge with the same weight
          const int64_t *b0 = indices + indptr[j], *b1 = indices + indptr[j + 1];
          const int64_t *it = std::lower_bound(b0, b1, i);
          if (it == b1 || *it != i || w[indptr[j] + (it - b0)] != w[p]) {
            bad[q] = i, why[q] = "half-edge (" + std::to_string(i) + ", " + std::to_string(j) +
                                 ") has no matching (" + std::to_string(j) + ", " +
                                 std::to_string(i) + ")";
            return;
          }
        }
      }
    });
  for (auto &x : th) x.join();
  for (int q = 0; q < t; ++q)
    if (bad[q] != INT64_MAX) throw Error(MG_ERR_INPUT, std::string(path) + ": " + why[q]);
}

}  // namespace mg
