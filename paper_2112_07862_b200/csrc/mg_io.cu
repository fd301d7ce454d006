// Text I/O either side of the path: the reference's CSV
// embedding writer/reader (embedding.py:131-166) and edge-list writer/reader
// (graph.py:147-196), byte-for-byte the same text, in multi-threaded C++.
//
// At config 5 the reference writes 20M rows x 32 coordinates through
// format(v, '.17g') one value at a time (~12 GB of text); here rows are
// formatted in parallel with std::to_chars (general, precision 17: the same
// correctly rounded digits as Python's '.17g') and written in order.  The
// readers parse with std::from_chars (correctly rounded, like float()) over
// line ranges in parallel and report the FIRST offending line, as the
// reference's sequential loop does.  Host-only code: no device work here.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mg_common.cuh"
#include "mg_io.cuh"

namespace mg {

namespace {

int pick_threads(int req) {
  int hw = (int)std::thread::hardware_concurrency();
  if (hw <= 0) hw = 1;
  return std::max(1, req > 0 ? std::min(req, 64) : std::min(hw, 32));
}

template <typename F>
void parallel_for(int64_t n, int threads, F f) {  // f(lo, hi, t)
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (T == 1) {
    f((int64_t)0, n, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([=]() { f(n * t / T, n * (t + 1) / T, t); });
  for (auto &th : pool) th.join();
}

// format(x, '.17g')
inline char *put_g17(char *p, char *end, double x) {
  auto r = std::to_chars(p, end, x, std::chars_format::general, 17);
  return r.ptr;
}
// str(float) (shortest round trip, '.0' for integral values)
std::string py_str(double x) {
  char b[64];
  auto r = std::to_chars(b, b + 64, x);
  std::string s(b, r.ptr);
  if (s.find_first_of(".en") == std::string::npos) s += ".0";
  return s;
}
// repr(str) for the ASCII lines of these files: single quotes unless the
// text holds one (then double quotes), backslash-escaped like Python
std::string py_repr(const std::string &s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = dq ? '"' : '\'';
  std::string o(1, q);
  for (char c : s) {
    if (c == '\\' || c == q) o += '\\';
    if (c == '\t') {
      o += "\\t";
      continue;
    }
    o += c;
  }
  return o + q;
}

bool read_file(const char *path, std::string &buf, std::string &err) {
  FILE *f = fopen(path, "rb");
  if (!f) {
    err = std::string("cannot open ") + path + ": [Errno " + std::to_string(errno) + "] " +
          strerror(errno) + ": '" + path + "'";
    return false;
  }
  fseek(f, 0, SEEK_END);
  const long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(&buf[0], 1, (size_t)sz, f) : 0;
  fclose(f);
  buf.resize(got);
  return true;
}

// line starts (universal newlines are not needed: the writers emit '\n')
void split_lines(const std::string &buf, std::vector<int64_t> &start) {
  start.clear();
  const int64_t n = (int64_t)buf.size();
  if (n == 0) return;
  start.push_back(0);
  const char *p = buf.data();
  for (int64_t i = 0; i < n; ++i)
    if (p[i] == '\n' && i + 1 < n) start.push_back(i + 1);
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\f' || c == '\v'; }

std::string strip(const char *b, const char *e) {
  while (b < e && is_ws(*b)) ++b;
  while (e > b && is_ws(e[-1])) --e;
  return std::string(b, e);
}

// int(s) / float(s) on a field (surrounding whitespace allowed, '+' sign ok)
bool parse_i64(const std::string &f0, int64_t &v) {
  std::string f = strip(f0.data(), f0.data() + f0.size());
  const char *b = f.data(), *e = b + f.size();
  if (b < e && *b == '+') ++b;
  if (b == e) return false;
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}
bool parse_f64(const std::string &f0, double &v) {
  std::string f = strip(f0.data(), f0.data() + f0.size());
  const char *b = f.data(), *e = b + f.size();
  if (b < e && *b == '+') ++b;
  if (b == e) return false;
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}

struct LineErr {
  int64_t line = -1;  // 0-based index into the line table, -1 = none
  int code = MG_OK;
  std::string msg;
};

}  // namespace

// ------------------------------------------------------------- embedding ---
void save_embedding_csv(const char *path, int64_t n, int k, const double *P, int threads) {
  require(path != nullptr && (n == 0 || P != nullptr) && k >= 0 && n >= 0, MG_ERR_INPUT,
          "bad embedding arguments");
  FILE *f = fopen(path, "wb");
  require(f != nullptr, MG_ERR_INPUT, std::string("cannot open ") + path + " for writing");
  std::string head = "node";
  for (int j = 0; j < k; ++j) head += ",c" + std::to_string(j + 1);
  head += "\n";
  fwrite(head.data(), 1, head.size(), f);
  const int T = pick_threads(threads);
  const int64_t chunk = 1 << 16;  // rows per formatted block
  std::vector<std::string> out(T);
  for (int64_t r0 = 0; r0 < n; r0 += chunk * T) {
    parallel_for(T, T, [&](int64_t lo, int64_t hi, int) {
      for (int64_t t = lo; t < hi; ++t) {
        std::string &s = out[t];
        s.clear();
        const int64_t a = r0 + t * chunk, b = std::min(n, a + chunk);
        if (a >= b) continue;
        s.resize((size_t)(b - a) * (size_t)(21 + 26 * (size_t)k));
        char *p = &s[0], *end = p + s.size();
        for (int64_t i = a; i < b; ++i) {
          p = std::to_chars(p, end, i).ptr;
          for (int j = 0; j < k; ++j) {
            *p++ = ',';
            p = put_g17(p, end, P[i * k + j]);
          }
          *p++ = '\n';
        }
        s.resize(p - &s[0]);
      }
    });
    for (int t = 0; t < T; ++t) fwrite(out[t].data(), 1, out[t].size(), f);
  }
  const bool ok = fclose(f) == 0;
  require(ok, MG_ERR_INPUT, std::string("write failed: ") + path);
}

void load_embedding_csv(const char *path, int64_t *n_out, int *k_out, double *P, int threads) {
  std::string buf, err;
  require(read_file(path, buf, err), MG_ERR_INPUT, err);
  std::vector<int64_t> st;
  split_lines(buf, st);
  const std::string p = path;
  auto line_of = [&](int64_t l) {
    const int64_t b = st[l], e = l + 1 < (int64_t)st.size() ? st[l + 1] : (int64_t)buf.size();
    return std::string(buf.data() + b, buf.data() + e);
  };
  // header: fh.readline().strip().split(",")
  std::vector<std::string> header;
  {
    const std::string h0 = st.empty() ? std::string() : line_of(0);
    const std::string h = strip(h0.data(), h0.data() + h0.size());
    size_t a = 0;
    while (true) {
      size_t c = h.find(',', a);
      header.push_back(h.substr(a, c == std::string::npos ? std::string::npos : c - a));
      if (c == std::string::npos) break;
      a = c + 1;
    }
  }
  require(!header.empty() && header[0] == "node", MG_ERR_INPUT,
          p + ": expected 'node,c1,...' header");
  const int k = (int)header.size() - 1;
  const int64_t n = st.empty() ? 0 : (int64_t)st.size() - 1;
  *n_out = n;
  *k_out = k;
  if (!P) return;  // dimension query
  std::vector<int64_t> ids(n);
  const int T = pick_threads(threads);
  std::vector<LineErr> errs(T);
  std::vector<double> rows((size_t)n * k);
  parallel_for(n, T, [&](int64_t lo, int64_t hi, int t) {
    for (int64_t r = lo; r < hi; ++r) {
      const std::string raw = line_of(r + 1);
      const std::string s = strip(raw.data(), raw.data() + raw.size());
      // line.strip().split(",")
      std::vector<std::string> parts;
      size_t a = 0;
      while (true) {
        size_t c = s.find(',', a);
        parts.push_back(s.substr(a, c == std::string::npos ? std::string::npos : c - a));
        if (c == std::string::npos) break;
        a = c + 1;
      }
      LineErr &E = errs[t];
      if (parts.size() != header.size()) {
        E = {r, MG_ERR_INPUT, p + ": ragged row " + py_repr(s)};
        return;
      }
      if (!parse_i64(parts[0], ids[r])) {
        E = {r, MG_ERR_INPUT,
             p + ": malformed embedding CSV: invalid literal for int() with base 10: " +
                 py_repr(parts[0])};
        return;
      }
      for (int j = 0; j < k; ++j)
        if (!parse_f64(parts[j + 1], rows[(size_t)r * k + j])) {
          E = {r, MG_ERR_INPUT,
               p + ": malformed embedding CSV: could not convert string to float: " +
                   py_repr(parts[j + 1])};
          return;
        }
    }
  });
  const LineErr *first = nullptr;
  for (auto &E : errs)
    if (E.line >= 0 && (!first || E.line < first->line)) first = &E;
  if (first) throw Error(first->code, first->msg);
  // ids must be a permutation of 0..n-1; P[order] puts row `id` at `id`
  std::vector<char> seen(n, 0);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t id = ids[r];
    require(id >= 0 && id < n && !seen[id], MG_ERR_INPUT, p + ": node ids must be dense 0..n-1");
    seen[id] = 1;
  }
  parallel_for(n, T, [&](int64_t lo, int64_t hi, int) {
    for (int64_t r = lo; r < hi; ++r)
      std::memcpy(P + ids[r] * k, rows.data() + (size_t)r * k, sizeof(double) * k);
  });
}

// ------------------------------------------------------------- edge list ---
void save_edge_list(const char *path, int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *w, int threads) {
  FILE *f = fopen(path, "wb");
  require(f != nullptr, MG_ERR_INPUT, std::string("cannot open ") + path + " for writing");
  const int T = pick_threads(threads);
  const int64_t chunk = 1 << 16;
  std::vector<std::string> out(T);
  for (int64_t r0 = 0; r0 < n; r0 += chunk * T) {
    parallel_for(T, T, [&](int64_t lo, int64_t hi, int) {
      for (int64_t t = lo; t < hi; ++t) {
        std::string &s = out[t];
        s.clear();
        const int64_t a = r0 + t * chunk, b = std::min(n, a + chunk);
        if (a >= b) continue;
        s.resize((size_t)(indptr[b] - indptr[a]) * 64 + 64);
        char *p = &s[0], *end = p + s.size();
        for (int64_t i = a; i < b; ++i)
          for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            if (!(i < indices[e])) continue;  // edge_array: rows < indices
            p = std::to_chars(p, end, i).ptr;
            *p++ = '\t';
            p = std::to_chars(p, end, indices[e]).ptr;
            *p++ = '\t';
            p = put_g17(p, end, w[e]);
            *p++ = '\n';
          }
        s.resize(p - &s[0]);
      }
    });
    for (int t = 0; t < T; ++t) fwrite(out[t].data(), 1, out[t].size(), f);
  }
  const bool ok = fclose(f) == 0;
  require(ok, MG_ERR_INPUT, std::string("write failed: ") + path);
}

void load_edge_list(const char *path, int threads, EdgeListResult &res) {
  std::string buf, err;
  require(read_file(path, buf, err), MG_ERR_INPUT, err);
  std::vector<int64_t> st;
  split_lines(buf, st);
  const std::string p = path;
  const int64_t L = (int64_t)st.size();
  const int T = pick_threads(threads);
  std::vector<LineErr> errs(T);
  // per line: kept flag + parsed edge
  std::vector<int64_t> ei(L, -1), ej(L, -1);
  std::vector<double> ew(L, 0.0);
  std::vector<char> keep(L, 0);
  parallel_for(L, T, [&](int64_t lo, int64_t hi, int t) {
    for (int64_t l = lo; l < hi; ++l) {
      const int64_t b = st[l], e = l + 1 < L ? st[l + 1] : (int64_t)buf.size();
      const std::string s = strip(buf.data() + b, buf.data() + e);
      if (s.empty() || s[0] == '#') continue;
      std::vector<std::string> parts;  // str.split(): whitespace runs
      size_t a = 0;
      while (a < s.size()) {
        while (a < s.size() && is_ws(s[a])) ++a;
        size_t c = a;
        while (c < s.size() && !is_ws(s[c])) ++c;
        if (c > a) parts.push_back(s.substr(a, c - a));
        a = c;
      }
      LineErr &E = errs[t];
      const std::string at = p + ":" + std::to_string(l + 1) + ": ";
      if (parts.size() != 2 && parts.size() != 3) {
        E = {l, MG_ERR_PARSE, at + "expected 'i j [w]', got " + py_repr(s)};
        return;
      }
      int64_t i, j;
      if (!parse_i64(parts[0], i) || !parse_i64(parts[1], j)) {
        E = {l, MG_ERR_PARSE, at + "node ids must be integers: " + py_repr(s)};
        return;
      }
      double w = 1.0;
      if (parts.size() == 3 && !parse_f64(parts[2], w)) {
        E = {l, MG_ERR_PARSE, at + "weight must be a number: " + py_repr(parts[2])};
        return;
      }
      if (i == j) {
        E = {l, MG_ERR_PARSE, at + "self-loop on node " + std::to_string(i)};
        return;
      }
      if (i < 0 || j < 0) {
        E = {l, MG_ERR_PARSE, at + "negative node id"};
        return;
      }
      if (!(w > 0.0)) {
        E = {l, MG_ERR_PARSE, at + "non-positive weight " + py_str(w)};
        return;
      }
      ei[l] = i;
      ej[l] = j;
      ew[l] = w;
      keep[l] = 1;
    }
  });
  const LineErr *first = nullptr;
  for (auto &E : errs)
    if (E.line >= 0 && (!first || E.line < first->line)) first = &E;
  if (first) {
    res.err_line = first->line + 1;
    throw Error(first->code, first->msg);
  }
  // Graph.from_edges (graph.py:31-79): n = max id + 1, duplicates rejected,
  // both half-edges bucketed by row, columns ascending
  int64_t E = 0, n = 0;
  for (int64_t l = 0; l < L; ++l)
    if (keep[l]) {
      ++E;
      n = std::max(n, std::max(ei[l], ej[l]) + 1);
    }
  require(E > 0, MG_ERR_INPUT, p + ": no edges");
  res.n = n;
  res.indptr.assign(n + 1, 0);
  for (int64_t l = 0; l < L; ++l)
    if (keep[l]) {
      ++res.indptr[ei[l] + 1];
      ++res.indptr[ej[l] + 1];
    }
  for (int64_t i = 0; i < n; ++i) res.indptr[i + 1] += res.indptr[i];
  std::vector<int64_t> fill(res.indptr.begin(), res.indptr.end() - 1);
  res.indices.resize(2 * E);
  res.weights.resize(2 * E);
  std::vector<int64_t> pos(2 * E);  // original (lo, hi) key for the duplicate message order
  for (int64_t l = 0; l < L; ++l)
    if (keep[l]) {
      int64_t q = fill[ei[l]]++;
      res.indices[q] = ej[l];
      res.weights[q] = ew[l];
      q = fill[ej[l]]++;
      res.indices[q] = ei[l];
      res.weights[q] = ew[l];
    }
  // sort each row by column (stable: equal columns = duplicates, rejected)
  std::vector<int64_t> dup_key(T, INT64_MAX);
  parallel_for(n, T, [&](int64_t lo, int64_t hi, int t) {
    std::vector<std::pair<int64_t, double>> row;
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t a = res.indptr[i], b = res.indptr[i + 1];
      row.clear();
      for (int64_t q = a; q < b; ++q) row.emplace_back(res.indices[q], res.weights[q]);
      std::stable_sort(row.begin(), row.end(),
                       [](const auto &x, const auto &y) { return x.first < y.first; });
      for (int64_t q = a; q < b; ++q) {
        res.indices[q] = row[q - a].first;
        res.weights[q] = row[q - a].second;
        if (q > a && res.indices[q] == res.indices[q - 1]) {
          const int64_t lo2 = std::min(i, res.indices[q]), hi2 = std::max(i, res.indices[q]);
          dup_key[t] = std::min(dup_key[t], lo2 * n + hi2);
        }
      }
    }
  });
  const int64_t dk = *std::min_element(dup_key.begin(), dup_key.end());
  require(dk == INT64_MAX, MG_ERR_INPUT,
          p + ": duplicate edge {" + std::to_string(dk / std::max<int64_t>(n, 1)) + ", " +
              std::to_string(dk % std::max<int64_t>(n, 1)) + "}");
}

}  // namespace mg
