// Tensor-file ingest for the sparse path: a multithreaded
// parser of the reference's `%rescalk-coo` text format straight into
// canonical per-slice CSR arrays.
//
// Reference: tensor.py:260-300 (_load_sparse: a pure-Python line loop, then
// scipy csr_matrix((vals, (rows, cols))) per slice) and the SparseRelTensor
// canonical form, tensor.py:96-104 (sum_duplicates, sort_indices,
// eliminate_zeros). Same acceptance rules and error texts:
//   line 1: "%rescalk-coo n m nnz"        -> "malformed header: ..."
//   data lines "t i j value" (blank lines skipped), 1-based line numbers:
//     wrong field count   -> "line L: expected 't i j value'"
//     unparsable field     -> "line L: ..."
//     t outside [0, m)     -> "line L: relation index t out of bounds"
//     (i, j) outside [0,n) -> "line L: index (i,j) out of bounds"
//     value < 0            -> "line L: negative value v"
//   entry count != nnz    -> "dimension mismatch: header says nnz=N, found C"
// The first failing line in file order is reported, as the sequential
// reference does. Values parse with std::from_chars (correctly rounded, like
// Python's float()); duplicates of one (t, i, j) are summed in file order
// (scipy sums them in std::sort order, which is unspecified for equal keys:
// bit-identical for up to two duplicates), then explicit zeros are dropped.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rescal_b200.h"

namespace {

struct Entry {
  int64_t key;  // (t * n + i) * n + j
  double v;
};

struct CooFile {
  int64_t n = 0, m = 0, nnz = 0;
  std::vector<int64_t> ptr;  // [m][n+1], per-slice offsets (start at 0)
  std::vector<int64_t> base; // first entry of slice t in idx/val
  std::vector<int32_t> idx;
  std::vector<double> val;
};

thread_local std::string g_err;

bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// Python int(): optional sign, decimal digits (leading zeros allowed)
bool parse_int(const char* b, const char* e, int64_t& out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b == e) return false;
  uint64_t v = 0;
  auto r = std::from_chars(b, e, v);
  if (r.ec != std::errc() || r.ptr != e || v > (uint64_t)INT64_MAX) return false;
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

// Python float(): optional sign, decimal / exponent forms, inf/infinity/nan
bool parse_float(const char* b, const char* e, double& out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b == e || *b == '+' || *b == '-') return false;
  auto r = std::from_chars(b, e, out);
  if (r.ec != std::errc() || r.ptr != e) return false;
  if (neg) out = -out;
  return true;
}

// Python repr() of a float (for the error texts): shortest round-trip digits,
// fixed notation for decimal exponents in [-4, 16), scientific otherwise.
std::string fmt_double(double v) {
  if (v != v) return "nan";
  if (v == 1.0 / 0.0) return "inf";
  if (v == -1.0 / 0.0) return "-inf";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  std::string s(buf, r.ptr);
  std::string sign;
  if (!s.empty() && s[0] == '-') {
    sign = "-";
    s = s.substr(1);
  }
  const size_t epos = s.find('e');
  std::string mant = s.substr(0, epos);
  const int ex = std::stoi(s.substr(epos + 1));
  std::string digits;
  for (char c : mant)
    if (c != '.') digits += c;
  if (ex >= -4 && ex < 16) {
    std::string out;
    if (ex < 0) {
      out = "0." + std::string((size_t)(-ex - 1), '0') + digits;
    } else if ((int)digits.size() <= ex + 1) {
      out = digits + std::string((size_t)(ex + 1 - (int)digits.size()), '0') + ".0";
    } else {
      out = digits.substr(0, (size_t)ex + 1) + "." + digits.substr((size_t)ex + 1);
    }
    return sign + out;
  }
  std::string out = digits.substr(0, 1);
  if (digits.size() > 1) out += "." + digits.substr(1);
  char eb[16];
  std::snprintf(eb, sizeof(eb), "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
  return sign + out + eb;
}

struct ChunkResult {
  std::vector<Entry> entries;
  int64_t lines = 0;        // newline-terminated lines in the chunk
  int64_t err_line = -1;    // chunk-local line index of the first error
  std::string err;
};

void parse_chunk(const char* b, const char* e, int64_t n, int64_t m, ChunkResult& res) {
  int64_t local = 0;
  const char* p = b;
  while (p < e) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
    const char* le = eol ? eol : e;
    const char* tok[5];
    const char* tend[5];
    int nt = 0;
    const char* q = p;
    while (q < le) {
      while (q < le && is_ws(*q)) ++q;
      if (q >= le) break;
      const char* s = q;
      while (q < le && !is_ws(*q)) ++q;
      if (nt < 5) {
        tok[nt] = s;
        tend[nt] = q;
      }
      ++nt;
    }
    if (nt != 0 && res.err_line < 0) {
      if (nt != 4) {
        res.err_line = local;
        res.err = "expected 't i j value'";
      } else {
        int64_t t, i, j;
        double v;
        if (!parse_int(tok[0], tend[0], t) || !parse_int(tok[1], tend[1], i) || !parse_int(tok[2], tend[2], j)) {
          res.err_line = local;
          res.err = "invalid literal for int()";
        } else if (!parse_float(tok[3], tend[3], v)) {
          res.err_line = local;
          res.err = "could not convert string to float: '" + std::string(tok[3], tend[3]) + "'";
        } else if (!(0 <= t && t < m)) {
          res.err_line = local;
          res.err = "relation index " + std::to_string(t) + " out of bounds";
        } else if (!(0 <= i && i < n && 0 <= j && j < n)) {
          res.err_line = local;
          res.err = "index (" + std::to_string(i) + "," + std::to_string(j) + ") out of bounds";
        } else if (v < 0) {
          res.err_line = local;
          res.err = "negative value " + fmt_double(v);
        } else {
          res.entries.push_back(Entry{(t * n + i) * n + j, v});
        }
      }
    }
    ++local;
    p = eol ? eol + 1 : e;
  }
  res.lines = local;
}

}  // namespace

extern "C" {

struct rk_coo {
  CooFile f;
};

int rk_coo_open(const char* path, rk_coo** out, int64_t* n_out, int64_t* m_out, int64_t* nnz_out) {
  static const bool timing = std::getenv("RK_UPLOAD_TIMING") != nullptr;  // diagnostics only
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rk] coo %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  try {
    if (!path || !out) throw std::string("null argument");
    *out = nullptr;
    FILE* fp = std::fopen(path, "rb");
    if (!fp) throw std::string("cannot open ") + path;
    std::fseek(fp, 0, SEEK_END);
    const long sz = std::ftell(fp);
    std::fseek(fp, 0, SEEK_SET);
    std::vector<char> buf((size_t)std::max(0L, sz));
    const size_t got = sz > 0 ? std::fread(buf.data(), 1, (size_t)sz, fp) : 0;
    std::fclose(fp);
    if ((long)got != sz) throw std::string("short read on ") + path;
    lap("read");
    const char* b = buf.data();
    const char* e = b + buf.size();
    // header (first line)
    const char* h_end = static_cast<const char*>(std::memchr(b, '\n', buf.size()));
    if (!h_end) h_end = e;
    std::vector<std::pair<const char*, const char*>> ht;
    for (const char* q = b; q < h_end;) {
      while (q < h_end && is_ws(*q)) ++q;
      if (q >= h_end) break;
      const char* s = q;
      while (q < h_end && !is_ws(*q)) ++q;
      ht.emplace_back(s, q);
    }
    if (ht.size() != 4 || std::string(ht[0].first, ht[0].second) != "%rescalk-coo")
      throw std::string("malformed header: expected '%rescalk-coo n m nnz'");
    int64_t n, m, nnz;
    if (!parse_int(ht[1].first, ht[1].second, n) || !parse_int(ht[2].first, ht[2].second, m) ||
        !parse_int(ht[3].first, ht[3].second, nnz))
      throw std::string("malformed header: invalid literal for int()");
    if (n < 0 || m < 0) throw std::string("malformed header: negative dimension");
    if (n >= (1ll << 31)) throw std::string("malformed header: n must fit int32 column indices");
    // data chunks split at newlines, parsed in parallel
    const char* d0 = h_end < e ? h_end + 1 : e;
    const unsigned hw = std::thread::hardware_concurrency();
    const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(hw ? hw : 1, (e - d0) / (1 << 20) + 1));
    std::vector<const char*> cut(nth + 1);
    cut[0] = d0;
    cut[nth] = e;
    for (int k = 1; k < nth; ++k) {
      const char* c = d0 + (e - d0) * k / nth;
      if (c < cut[k - 1]) c = cut[k - 1];
      const char* nl = c < e ? static_cast<const char*>(std::memchr(c, '\n', (size_t)(e - c))) : nullptr;
      cut[k] = nl ? nl + 1 : e;
    }
    std::vector<ChunkResult> res(nth);
    {
      std::vector<std::thread> th;
      for (int k = 0; k < nth; ++k)
        th.emplace_back([&, k] { parse_chunk(cut[k], cut[k + 1], n, m, res[k]); });
      for (auto& t : th) t.join();
    }
    lap("parse");
    int64_t line0 = 2, count = 0;
    for (int k = 0; k < nth; ++k) {
      if (res[k].err_line >= 0)
        throw "line " + std::to_string(line0 + res[k].err_line) + ": " + res[k].err;
      line0 += res[k].lines;
      count += (int64_t)res[k].entries.size();
    }
    if (count != nnz)
      throw "dimension mismatch: header says nnz=" + std::to_string(nnz) + ", found " + std::to_string(count);
    // canonical CSR: stable order by (t, i, j) (file order among duplicates),
    // duplicates summed, zeros dropped
    // files written by save_tensor are in (t, i, j) order (tensor.py:249-257):
    // then no sort is needed; otherwise a stable sort keeps file order among
    // duplicates
    bool sorted = true;
    int64_t last = -1;
    for (auto& r : res) {
      for (const Entry& en : r.entries) {
        if (en.key < last) {
          sorted = false;
          break;
        }
        last = en.key;
      }
      if (!sorted) break;
    }
    std::vector<Entry> all;
    all.reserve((size_t)count);
    for (auto& r : res) {
      all.insert(all.end(), r.entries.begin(), r.entries.end());
      std::vector<Entry>().swap(r.entries);
    }
    lap("concat");
    if (!sorted)
      std::stable_sort(all.begin(), all.end(), [](const Entry& a, const Entry& c) { return a.key < c.key; });
    auto* h = new rk_coo();
    CooFile& f = h->f;
    f.n = n;
    f.m = m;
    f.ptr.assign((size_t)m * (n + 1), 0);
    f.base.assign((size_t)m + 1, 0);
    f.idx.reserve(all.size());
    f.val.reserve(all.size());
    std::vector<int64_t> key_of;
    key_of.reserve(all.size());
    for (size_t a = 0; a < all.size();) {
      size_t c = a + 1;
      double s = all[a].v;
      while (c < all.size() && all[c].key == all[a].key) s += all[c++].v;
      if (s != 0.0) {
        key_of.push_back(all[a].key);
        f.val.push_back(s);
      }
      a = c;
    }
    std::vector<Entry>().swap(all);
    f.idx.resize(key_of.size());
    for (size_t q = 0; q < key_of.size(); ++q) {
      const int64_t key = key_of[q];
      const int64_t t = key / (n * n), i = (key / n) % n, j = key % n;
      f.idx[q] = (int32_t)j;
      f.ptr[(size_t)t * (n + 1) + i + 1] += 1;
      f.base[(size_t)t + 1] += 1;
    }
    for (int64_t t = 0; t < m; ++t) {
      int64_t* pt = f.ptr.data() + (size_t)t * (n + 1);
      for (int64_t i = 0; i < n; ++i) pt[i + 1] += pt[i];
      f.base[(size_t)t + 1] += f.base[(size_t)t];
    }
    f.nnz = (int64_t)key_of.size();
    lap("csr");
    *out = h;
    if (n_out) *n_out = n;
    if (m_out) *m_out = m;
    if (nnz_out) *nnz_out = f.nnz;
    return RK_OK;
  } catch (const std::string& msg) {
    g_err = msg;
    return RK_ERR_DATA;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return RK_ERR_DATA;
  }
}

const char* rk_coo_last_error(void) { return g_err.c_str(); }

int64_t rk_coo_slice_nnz(const rk_coo* h, int64_t t) {
  if (!h || t < 0 || t >= h->f.m) return -1;
  return h->f.base[(size_t)t + 1] - h->f.base[(size_t)t];
}

int rk_coo_fill(const rk_coo* h, int64_t t, int64_t* indptr, int32_t* indices, double* data) {
  if (!h || t < 0 || t >= h->f.m || !indptr) return RK_ERR_DATA;
  const CooFile& f = h->f;
  std::memcpy(indptr, f.ptr.data() + (size_t)t * (f.n + 1), sizeof(int64_t) * (f.n + 1));
  const int64_t b = f.base[(size_t)t], c = f.base[(size_t)t + 1] - b;
  if (c > 0) {
    if (!indices || !data) return RK_ERR_DATA;
    std::memcpy(indices, f.idx.data() + b, sizeof(int32_t) * c);
    std::memcpy(data, f.val.data() + b, sizeof(double) * c);
  }
  return RK_OK;
}

void rk_coo_close(rk_coo* h) { delete h; }

}  // extern "C"
