// Edge-list text I/O on the host, multi-threaded (reference graph.py:177-225).
//
// read: the file is read once and split into per-thread chunks at '\n' boundaries; every
// line is classified exactly as the reference's loop does (graph.py:188-210, text mode with
// universal newlines, str.strip / str.split on ASCII whitespace):
//   blank -> skipped; '#' -> comment, "# nodes N" sets the header node count (last wins);
//   otherwise 2 or 3 tokens "src dst [weight]" -> one row (weight 1.0 when absent).
// Tokens are parsed natively only on a grammar whose value provably equals Python's
// int() / float() ([+-]?digits for ints up to 18 digits; decimal floats, correctly rounded
// by std::from_chars like CPython's dtoa).  A line outside that grammar (any non-ASCII
// byte, underscores, inf/nan, overflow, a wrong token count, ...) is reported as *complex*
// with its line number and byte range, and a row slot is reserved for it when it is a data
// line: the Python caller re-parses exactly those lines with the reference's own rules, so
// values, row order and the first error raised are the reference's.
//
// write: one "i j repr(w)\n" line per stored entry with i < j in CSR order (the order of
// W.tocoo() in graph.py:218-225), after a "# nodes N" header; repr() is Python's shortest
// round-trip float formatting, rebuilt from std::to_chars' shortest digits.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace csc {
namespace {

inline bool is_ws(unsigned char c) {  // str.isspace() on ASCII
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// [+-]?[0-9]{1,18}: exactly Python's int() on that grammar
bool parse_int(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b == e || e - b > 18) return false;
  int64_t v = 0;
  for (const char* p = b; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (*p - '0');
  }
  *out = neg ? -v : v;
  return true;
}

// [+-]?(digits[.digits*]|.digits)([eE][+-]?digits)?, finite and in range: Python's float()
bool parse_float(const char* b, const char* e, double* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  const char* p = b;
  int mant = 0;
  while (p < e && *p >= '0' && *p <= '9') ++p, ++mant;
  if (p < e && *p == '.') {
    ++p;
    while (p < e && *p >= '0' && *p <= '9') ++p, ++mant;
  }
  if (mant == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    int ed = 0;
    while (p < e && *p >= '0' && *p <= '9') ++p, ++ed;
    if (ed == 0) return false;
  }
  if (p != e) return false;
  double v = 0.0;
  const auto r = std::from_chars(b, e, v, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr != e) return false;  // out of range: Python gives inf / 0
  *out = neg ? -v : v;
  return true;
}

struct Complex {
  int64_t line;    // 1-based line number (chunk-local until merged)
  int64_t slot;    // reserved row slot (chunk-local until merged), -1 for comment lines
  int64_t offset;  // byte offset of the line in the file
  int64_t length;  // bytes, without the line terminator
};

struct Chunk {
  const char* b = nullptr;
  const char* e = nullptr;
  int64_t lines = 0;
  std::vector<double> src, dst, w;
  std::vector<uint8_t> cx;  // per row: 1 = complex placeholder
  std::vector<Complex> complex;
  int64_t header_nodes = -1, header_line = 0;
};

void parse_chunk(Chunk& c, const char* base) {
  const char* p = c.b;
  int64_t ln = 0;
  while (p < c.e) {
    const char* t = p;
    while (t < c.e && *t != '\n' && *t != '\r') ++t;
    const char* next = t;
    if (next < c.e) next += (*next == '\r' && next + 1 < c.e && next[1] == '\n') ? 2 : 1;
    ++ln;
    const char* lb = p;
    const char* le = t;
    p = next;
    bool ascii = true;
    for (const char* q = lb; q < le; ++q)
      if ((unsigned char)*q >= 0x80) {
        ascii = false;
        break;
      }
    if (!ascii) {  // Python decides (utf-8 decoding, Unicode whitespace and digits); the slot is
                   // dropped by the caller if the line turns out blank or a comment
      c.complex.push_back({ln, (int64_t)c.src.size(), lb - base, le - lb});
      c.src.push_back(0.0), c.dst.push_back(0.0), c.w.push_back(0.0), c.cx.push_back(1);
      continue;
    }
    while (lb < le && is_ws((unsigned char)*lb)) ++lb;
    while (le > lb && is_ws((unsigned char)le[-1])) --le;
    if (lb == le) continue;  // blank
    // split into at most 4 tokens (4 means "too many")
    const char* tb[4];
    const char* te[4];
    int nt = 0;
    const char* q = (*lb == '#') ? lb + 1 : lb;
    while (q < le && nt < 4) {
      while (q < le && is_ws((unsigned char)*q)) ++q;
      if (q >= le) break;
      tb[nt] = q;
      while (q < le && !is_ws((unsigned char)*q)) ++q;
      te[nt++] = q;
    }
    if (*lb == '#') {  // comment; "# nodes N" (exactly two tokens) sets the header
      if (nt == 2 && te[0] - tb[0] == 5 && std::memcmp(tb[0], "nodes", 5) == 0) {
        int64_t v = 0;
        if (parse_int(tb[1], te[1], &v)) {
          c.header_nodes = v;
          c.header_line = ln;
        } else {
          c.complex.push_back({ln, -1, lb - base, le - lb});
        }
      }
      continue;
    }
    int64_t i = 0, j = 0;
    double w = 1.0;
    const bool ok = (nt == 2 || nt == 3) && parse_int(tb[0], te[0], &i) && parse_int(tb[1], te[1], &j) &&
                    (nt == 2 || parse_float(tb[2], te[2], &w));
    if (ok) {
      c.src.push_back((double)i), c.dst.push_back((double)j), c.w.push_back(w), c.cx.push_back(0);
    } else {
      c.complex.push_back({ln, (int64_t)c.src.size(), lb - base, le - lb});
      c.src.push_back(0.0), c.dst.push_back(0.0), c.w.push_back(0.0), c.cx.push_back(1);
    }
  }
  c.lines = ln;
}

int threads_for(int64_t bytes, int nthreads) {
  int t = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (t < 1) t = 1;
  const int64_t per = 4 << 20;  // >= 4 MB per thread
  if (bytes / per + 1 < t) t = (int)(bytes / per + 1);
  return t;
}

// Python repr(float): shortest round-trip digits; fixed notation when -4 < decpt <= 16
// (decpt = decimal exponent + 1), else d[.ddd]e[+-]XX with at least two exponent digits;
// fixed notation always shows a fractional part ("1.0").
int py_repr(double v, char* out) {
  char buf[64];
  if (v != v) return (int)(std::memcpy(out, "nan", 3), 3);
  int n = 0;
  if (std::signbit(v)) out[n++] = '-', v = -v;
  if (v == __builtin_inf()) return std::memcpy(out + n, "inf", 3), n + 3;
  if (v == 0.0) return std::memcpy(out + n, "0.0", 3), n + 3;
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  // buf: d[.ddd]e[+-]XX
  char digits[32];
  int nd = 0;
  const char* p = buf;
  for (; p < r.ptr && *p != 'e'; ++p)
    if (*p != '.') digits[nd++] = *p;
  int exp10 = 0;
  std::from_chars(p + 1 + (p[1] == '+' ? 1 : 0), r.ptr, exp10);
  const int decpt = exp10 + 1;
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      out[n++] = '0', out[n++] = '.';
      for (int k = 0; k < -decpt; ++k) out[n++] = '0';
      for (int k = 0; k < nd; ++k) out[n++] = digits[k];
    } else if (decpt < nd) {
      for (int k = 0; k < decpt; ++k) out[n++] = digits[k];
      out[n++] = '.';
      for (int k = decpt; k < nd; ++k) out[n++] = digits[k];
    } else {
      for (int k = 0; k < nd; ++k) out[n++] = digits[k];
      for (int k = nd; k < decpt; ++k) out[n++] = '0';
      out[n++] = '.', out[n++] = '0';
    }
    return n;
  }
  out[n++] = digits[0];
  if (nd > 1) {
    out[n++] = '.';
    for (int k = 1; k < nd; ++k) out[n++] = digits[k];
  }
  out[n++] = 'e';
  out[n++] = exp10 < 0 ? '-' : '+';
  const int ax = exp10 < 0 ? -exp10 : exp10;
  if (ax < 10) out[n++] = '0';
  const auto er = std::to_chars(out + n, out + n + 8, ax);
  return (int)(er.ptr - out);
}

}  // namespace
}  // namespace csc

struct csc_edges {
  std::vector<double> src, dst, w;
  std::vector<uint8_t> cx;
  std::vector<csc::Complex> complex;
  int64_t header_nodes = -1, header_line = 0;
};

using namespace csc;

extern "C" int csc_edgelist_read(const char* path, int nthreads, csc_edges** out) {
  return guard([&] {
    if (!path || !out) fail(CSC_ERR_INVALID, "path / out is NULL");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(CSC_ERR_INVALID, std::string("cannot open ") + path);
    std::fseek(f, 0, SEEK_END);
    const int64_t size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::string data((size_t)std::max<int64_t>(size, 0), '\0');
    const size_t got = size > 0 ? std::fread(&data[0], 1, (size_t)size, f) : 0;
    std::fclose(f);
    if ((int64_t)got != size) fail(CSC_ERR_INVALID, std::string("short read of ") + path);
    const char* base = data.data();
    const int T = threads_for(size, nthreads);
    std::vector<Chunk> ch(T);
    int64_t start = 0;
    for (int t = 0; t < T; ++t) {  // split after a '\n' (never inside "\r\n")
      int64_t stop = t == T - 1 ? size : std::max<int64_t>(start, size * (t + 1) / T);
      while (stop < size && stop > 0 && base[stop - 1] != '\n') ++stop;
      ch[t].b = base + start;
      ch[t].e = base + stop;
      start = stop;
    }
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(parse_chunk, std::ref(ch[t]), base);
    parse_chunk(ch[0], base);
    for (auto& th : pool) th.join();
    auto* e = new csc_edges();
    int64_t rows = 0, ncx = 0;
    for (auto& c : ch) rows += (int64_t)c.src.size(), ncx += (int64_t)c.complex.size();
    e->src.reserve(rows), e->dst.reserve(rows), e->w.reserve(rows), e->cx.reserve(rows);
    e->complex.reserve(ncx);
    int64_t line0 = 0, row0 = 0;
    for (auto& c : ch) {
      e->src.insert(e->src.end(), c.src.begin(), c.src.end());
      e->dst.insert(e->dst.end(), c.dst.begin(), c.dst.end());
      e->w.insert(e->w.end(), c.w.begin(), c.w.end());
      e->cx.insert(e->cx.end(), c.cx.begin(), c.cx.end());
      for (auto x : c.complex) {
        x.line += line0;
        if (x.slot >= 0) x.slot += row0;
        e->complex.push_back(x);
      }
      if (c.header_line > 0) e->header_nodes = c.header_nodes, e->header_line = c.header_line + line0;
      line0 += c.lines;
      row0 += (int64_t)c.src.size();
    }
    *out = e;
  });
}

extern "C" int csc_edgelist_info(const csc_edges* e, int64_t* num_rows, int64_t* num_complex, int64_t* header_nodes,
                                 int64_t* header_line) {
  return guard([&] {
    if (!e) fail(CSC_ERR_INVALID, "edge list is NULL");
    if (num_rows) *num_rows = (int64_t)e->src.size();
    if (num_complex) *num_complex = (int64_t)e->complex.size();
    if (header_nodes) *header_nodes = e->header_nodes;
    if (header_line) *header_line = e->header_line;
  });
}

extern "C" int csc_edgelist_rows(const csc_edges* e, double* src, double* dst, double* w, uint8_t* complex_row) {
  return guard([&] {
    if (!e) fail(CSC_ERR_INVALID, "edge list is NULL");
    const size_t n = e->src.size();
    if (n && (!src || !dst || !w)) fail(CSC_ERR_INVALID, "row arrays are NULL");
    if (n) {
      std::memcpy(src, e->src.data(), n * sizeof(double));
      std::memcpy(dst, e->dst.data(), n * sizeof(double));
      std::memcpy(w, e->w.data(), n * sizeof(double));
      if (complex_row) std::memcpy(complex_row, e->cx.data(), n);
    }
  });
}

extern "C" int csc_edgelist_complex(const csc_edges* e, int64_t* line_numbers, int64_t* row_slots,
                                    int64_t* byte_offsets, int64_t* byte_lengths) {
  return guard([&] {
    if (!e) fail(CSC_ERR_INVALID, "edge list is NULL");
    for (size_t k = 0; k < e->complex.size(); ++k) {
      if (line_numbers) line_numbers[k] = e->complex[k].line;
      if (row_slots) row_slots[k] = e->complex[k].slot;
      if (byte_offsets) byte_offsets[k] = e->complex[k].offset;
      if (byte_lengths) byte_lengths[k] = e->complex[k].length;
    }
  });
}

extern "C" int csc_edgelist_destroy(csc_edges* e) {
  return guard([&] { delete e; });
}

extern "C" int csc_edgelist_write(const char* path, int64_t num_nodes, const int32_t* indptr, const int32_t* indices,
                                  const double* weights, int nthreads) {
  return guard([&] {
    if (!path) fail(CSC_ERR_INVALID, "path is NULL");
    if (num_nodes < 0) fail(CSC_ERR_INVALID, "num_nodes < 0");
    if (num_nodes > 0 && !indptr) fail(CSC_ERR_INVALID, "indptr is NULL");
    const int64_t nnz = num_nodes > 0 ? indptr[num_nodes] : 0;
    if (nnz > 0 && (!indices || !weights)) fail(CSC_ERR_INVALID, "indices / weights are NULL");
    const int T = threads_for(nnz * 24, nthreads);
    std::vector<std::string> part(T);
    auto fmt = [&](int t) {
      const int64_t r0 = num_nodes * t / T, r1 = num_nodes * (t + 1) / T;
      std::string& s = part[t];
      if (r1 > r0) s.reserve((size_t)std::max<int64_t>(0, indptr[r1] - indptr[r0]) * 14);
      char line[96];
      for (int64_t i = r0; i < r1; ++i)
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
          const int64_t j = indices[k];
          if (i >= j) continue;
          char* p = std::to_chars(line, line + 24, i).ptr;
          *p++ = ' ';
          p = std::to_chars(p, p + 24, j).ptr;
          *p++ = ' ';
          p += py_repr(weights[k], p);
          *p++ = '\n';
          s.append(line, (size_t)(p - line));
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(fmt, t);
    fmt(0);
    for (auto& th : pool) th.join();
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(CSC_ERR_INVALID, std::string("cannot open ") + path + " for writing");
    const std::string head = "# nodes " + std::to_string(num_nodes) + "\n";
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    for (auto& s : part) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) fail(CSC_ERR_INVALID, std::string("write failed: ") + path);
  });
}

// Test hook: Python's repr() of a double as this library formats it.
extern "C" int csc_float_repr(double v, char* out, int cap, int* len) {
  return guard([&] {
    if (!out || cap < 32) fail(CSC_ERR_INVALID, "need a >= 32-byte buffer");
    const int n = py_repr(v, out);
    out[n] = '\0';
    if (len) *len = n;
  });
}
