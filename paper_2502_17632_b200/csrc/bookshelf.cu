// bookshelf.cu -- Bookshelf reader on the device.
//
// Reference: parse_design, giftplace/netlist.py:418-458, with the per-file
// parsers _data_lines :196-205, _header_value :208-212, _parse_nodes :215-250,
// _parse_nets :253-310, _parse_pl :313-327 and the error classes of
// errors.py (MalformedLineError, DuplicateCellError, DanglingPinError).
// The .aux manifest and the .scl rows are a few lines and stay on the host
// (paper_2502_17632_b200/bookshelf.py).
//
// The reference walks the files line by line in Python.  Here every line is
// independent work:
//   1. line starts (universal newlines: \n, \r\n, \r -- Python text mode),
//      comment cut at the first '#', whitespace strip, "UCLA" headers and
//      blank lines dropped  -> data lines with their 1-based line numbers;
//   2. one thread per data line tokenises it (Python str.split() whitespace)
//      and parses numbers exactly like float() / int();
//   3. the sequential parts of the reference become scans: cell ids are the
//      rank among cell lines, a pin line's net is the count of NetDegree
//      lines before it, its position in the net the pin rank minus the net's
//      first pin rank, and "pending" (the pin lines a NetDegree still
//      expects) is count - pins seen, so every error the reference raises is
//      attributed to a line;
//   4. the reference stops at the FIRST error in line order: that is the
//      minimum line over all per-line errors, with the reference's check
//      order inside one line kept (e.g. "previous net is missing" before a
//      NetDegree's own syntax);
//   5. names: 64-bit hashes, a radix sort finds duplicate cell names (the
//      later line is the DuplicateCellError, as in the reference), an
//      open-addressing table maps pin / .pl names to cell ids (bytes are
//      compared on a hash hit);
//   6. .pl: the last line naming a cell wins (the reference's dict
//      assignment), fixed = .nodes "terminal" or .pl /FIXED, fixed centre =
//      lower-left + size / 2, plus the placement bounding box for the
//      region fallback.
//
// Numbers: float() is the correctly rounded decimal value.  The device
// decides every token with <= 19 significant digits and a decimal exponent
// in [-22, 22] exactly (Clinger's fast path: both operands exact, one IEEE
// operation) and the grammar of every token; the rare rest (more digits,
// larger exponents, '_' separators) is re-parsed on the host from the
// caller's buffer with the same line parser and strtod (correctly rounded).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cerrno>
#include <climits>
#include <clocale>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <locale.h>
#include <string>
#include <vector>

#include "common.cuh"

namespace gift {
namespace bs {

// error codes (mirrored in paper_2502_17632_b200/bookshelf.py)
enum : int {
  E_OK = 0,
  N_HDR_COLON = 1, N_HDR_INT = 2, N_FEW = 3, N_NUM = 4, N_POS = 5, N_DUP = 6, N_COUNT = 7,
  T_HDR_COLON = 20, T_HDR_INT = 21, T_PREV_MISSING = 22, T_DEG_COLON = 23, T_DEG_INT = 24, T_OUTSIDE = 25,
  T_DANGLING = 26, T_OFFS = 27, T_LAST_MISSING = 28, T_COUNT = 29,
  P_FEW = 40, P_NUM = 41, P_NOPLACE = 42,
  X_UNICODE_WS = 60, X_INT_RANGE = 61, X_HASH = 62,
};

constexpr int kBlock = 256;

// ---- character classes / tokens (host + device) ----------------------------
__host__ __device__ __forceinline__ bool is_ws(unsigned char c) {
  // Python str.split()/strip() ASCII whitespace (\x1c-\x1f are separators too)
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// next whitespace-separated token in [pos, end): returns false when none
__host__ __device__ __forceinline__ bool next_tok(const char* s, int& pos, int end, int& tb, int& te) {
  while (pos < end && is_ws((unsigned char)s[pos])) ++pos;
  if (pos >= end) return false;
  tb = pos;
  while (pos < end && !is_ws((unsigned char)s[pos])) ++pos;
  te = pos;
  return true;
}

__host__ __device__ __forceinline__ bool tok_eq(const char* s, int b, int e, const char* lit) {
  int i = 0;
  for (; lit[i]; ++i)
    if (b + i >= e || s[b + i] != lit[i]) return false;
  return b + i == e;
}

__host__ __device__ __forceinline__ bool tok_starts(const char* s, int b, int e, const char* lit) {
  for (int i = 0; lit[i]; ++i)
    if (b + i >= e || s[b + i] != lit[i]) return false;
  return true;
}

__host__ __device__ __forceinline__ void strip(const char* s, int& b, int& e) {
  while (b < e && is_ws((unsigned char)s[b])) ++b;
  while (e > b && is_ws((unsigned char)s[e - 1])) --e;
}

__host__ __device__ __forceinline__ char lower(char c) { return (c >= 'A' && c <= 'Z') ? (char)(c + 32) : c; }

__host__ __device__ __forceinline__ bool word_ieq(const char* s, int b, int e, const char* lit) {
  int i = 0;
  for (; lit[i]; ++i)
    if (b + i >= e || lower(s[b + i]) != lit[i]) return false;
  return b + i == e;
}

// ---- Python int() / float() -------------------------------------------------
enum : int { NUM_OK = 0, NUM_BAD = 1, NUM_SLOW = 2, NUM_RANGE = 3 };

// int(): [sign] digits with single '_' between digits; int64 range
__host__ __device__ inline int py_int(const char* s, int b, int e, long long* out) {
  if (b >= e) return NUM_BAD;
  bool neg = false;
  if (s[b] == '+' || s[b] == '-') {
    neg = s[b] == '-';
    ++b;
  }
  if (b >= e) return NUM_BAD;
  unsigned long long v = 0;
  bool prev_digit = false, range = false;
  for (int i = b; i < e; ++i) {
    const char c = s[i];
    if (c >= '0' && c <= '9') {
      if (v > (ULLONG_MAX - 9) / 10) range = true;
      v = v * 10 + (unsigned)(c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < e && s[i + 1] >= '0' && s[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return NUM_BAD;
    }
  }
  if (range || v > (unsigned long long)LLONG_MAX + (neg ? 1ull : 0ull)) return NUM_RANGE;
  *out = neg ? (long long)(0ull - v) : (long long)v;
  return NUM_OK;
}

// float() grammar check; digits may carry '_' separators (PEP 515)
__host__ __device__ inline bool py_float_grammar(const char* s, int b, int e, bool* has_us) {
  *has_us = false;
  if (b < e && (s[b] == '+' || s[b] == '-')) ++b;
  if (b >= e) return false;
  if (word_ieq(s, b, e, "inf") || word_ieq(s, b, e, "infinity") || word_ieq(s, b, e, "nan")) return true;
  auto digits = [&](int& i) {  // digitpart: digit (['_'] digit)*, returns #digits
    int nd = 0;
    while (i < e) {
      if (s[i] >= '0' && s[i] <= '9') {
        ++nd;
        ++i;
      } else if (s[i] == '_' && nd > 0 && i + 1 < e && s[i + 1] >= '0' && s[i + 1] <= '9') {
        *has_us = true;
        ++i;
      } else {
        break;
      }
    }
    return nd;
  };
  int i = b;
  const int n_int = digits(i);
  int n_frac = 0;
  if (i < e && s[i] == '.') {
    ++i;
    n_frac = digits(i);
  }
  if (n_int == 0 && n_frac == 0) return false;
  if (i < e && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    if (i < e && (s[i] == '+' || s[i] == '-')) ++i;
    if (digits(i) == 0) return false;
  }
  return i == e;
}

__host__ __device__ __forceinline__ double pow10_exact(int k) {  // 10^k, k <= 22: exact
  double p = 1.0;
  for (int i = 0; i < k; ++i) p *= 10.0;
  return p;
}

// device decision: NUM_OK (exact), NUM_BAD (not a float), NUM_SLOW (host decides)
__host__ __device__ inline int py_float_fast(const char* s, int b, int e, double* out) {
  bool us = false;
  if (!py_float_grammar(s, b, e, &us)) return NUM_BAD;
  if (us) return NUM_SLOW;
  bool neg = false;
  if (s[b] == '+' || s[b] == '-') {
    neg = s[b] == '-';
    ++b;
  }
  if (word_ieq(s, b, e, "inf") || word_ieq(s, b, e, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return NUM_OK;
  }
  if (word_ieq(s, b, e, "nan")) {
    *out = neg ? -NAN : NAN;
    return NUM_OK;
  }
  unsigned long long m = 0;
  int nd = 0, frac = 0, i = b;
  bool point = false;
  for (; i < e && s[i] != 'e' && s[i] != 'E'; ++i) {
    if (s[i] == '.') {
      point = true;
      continue;
    }
    const int d = s[i] - '0';
    if (point) ++frac;
    if (m == 0 && d == 0) continue;  // leading zeros
    if (++nd > 19) return NUM_SLOW;
    m = m * 10 + (unsigned)d;
  }
  long long ex = 0;
  if (i < e) {
    ++i;
    bool eneg = false;
    if (s[i] == '+' || s[i] == '-') {
      eneg = s[i] == '-';
      ++i;
    }
    for (; i < e; ++i) {
      if (ex < 100000) ex = ex * 10 + (s[i] - '0');
    }
    if (eneg) ex = -ex;
  }
  if (m == 0) {
    *out = neg ? -0.0 : 0.0;
    return NUM_OK;
  }
  const long long k = ex - frac;
  if (m > (1ull << 53) || k < -22 || k > 22) return NUM_SLOW;
  double v = (double)m;  // exact
  v = k >= 0 ? v * pow10_exact((int)k) : v / pow10_exact((int)-k);
  *out = neg ? -v : v;
  return NUM_OK;
}

// host: the full float() (grammar above, then strtod in the C locale)
inline int py_float_host(const char* s, int b, int e, double* out) {
  const int r = py_float_fast(s, b, e, out);
  if (r != NUM_SLOW) return r;
  std::string t;
  t.reserve(e - b);
  for (int i = b; i < e; ++i)
    if (s[i] != '_') t.push_back(s[i]);
  static locale_t c_loc = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
  char* endp = nullptr;
  errno = 0;
  double v = strtod_l(t.c_str(), &endp, c_loc);
  if (endp != t.c_str() + t.size()) return NUM_BAD;
  *out = v;  // overflow -> +-inf, underflow -> correctly rounded subnormal / 0, as float()
  return NUM_OK;
}

template <bool HOST>
__host__ __device__ __forceinline__ int parse_float(const char* s, int b, int e, double* out) {
#ifdef __CUDA_ARCH__
  return py_float_fast(s, b, e, out);
#else
  return HOST ? py_float_host(s, b, e, out) : py_float_fast(s, b, e, out);
#endif
}

// ---- per-line records ---------------------------------------------------------
struct NodeRec {
  int kind;  // 0 cell, 1 NumNodes, 2 NumTerminals
  int err;
  int slow;
  int term;
  int nb, ne;  // name token, relative to the line start
  long long hval;
  double w, h;
};

struct NetRec {
  int kind;  // 1 NumNets, 2 NumPins, 3 NetDegree, 4 pin
  int err;
  int slow;
  int nb, ne;  // NetDegree name (ne < 0: none) or pin cell name
  long long val;
  double dx, dy;
};

struct PlRec {
  int err;
  int slow;
  int fixed;
  int nb, ne;
  double x, y;
};

// header value: text after the first ':' of the line, stripped (netlist.py:208-212)
__host__ __device__ __forceinline__ bool header_value(const char* s, int n, int& vb, int& ve) {
  int c = 0;
  while (c < n && s[c] != ':') ++c;
  if (c >= n) return false;
  vb = c + 1;
  ve = n;
  strip(s, vb, ve);
  return true;
}

template <bool HOST>
__host__ __device__ NodeRec parse_node_line(const char* s, int n) {  // netlist.py:215-250
  NodeRec r{};
  int pos = 0, tb = 0, te = 0;
  next_tok(s, pos, n, tb, te);
  const bool nn = tok_eq(s, tb, te, "NumNodes");
  if (nn || tok_eq(s, tb, te, "NumTerminals")) {
    r.kind = nn ? 1 : 2;
    int vb, ve;
    if (!header_value(s, n, vb, ve)) {
      r.err = N_HDR_COLON;
      return r;
    }
    const int q = py_int(s, vb, ve, &r.hval);
    if (q == NUM_BAD) r.err = N_HDR_INT;
    if (q == NUM_RANGE) r.err = X_INT_RANGE;
    return r;
  }
  r.nb = tb;
  r.ne = te;
  int b1, e1, b2, e2;
  if (!next_tok(s, pos, n, b1, e1) || !next_tok(s, pos, n, b2, e2)) {
    r.err = N_FEW;
    return r;
  }
  const int q1 = parse_float<HOST>(s, b1, e1, &r.w);
  if (q1 == NUM_SLOW) {
    r.slow = 1;
    return r;
  }
  if (q1 == NUM_BAD) {
    r.err = N_NUM;
    return r;
  }
  const int q2 = parse_float<HOST>(s, b2, e2, &r.h);
  if (q2 == NUM_SLOW) {
    r.slow = 1;
    return r;
  }
  if (q2 == NUM_BAD) {
    r.err = N_NUM;
    return r;
  }
  if (r.w <= 0 || r.h <= 0) {  // NaN passes, as in the reference
    r.err = N_POS;
    return r;
  }
  int b, e;
  while (next_tok(s, pos, n, b, e))
    if (tok_starts(s, b, e, "terminal")) r.term = 1;
  return r;
}

template <bool HOST>
__host__ __device__ NetRec parse_net_line(const char* s, int n) {  // netlist.py:253-310
  NetRec r{};
  int pos = 0, tb = 0, te = 0;
  next_tok(s, pos, n, tb, te);
  const bool nn = tok_eq(s, tb, te, "NumNets");
  if (nn || tok_eq(s, tb, te, "NumPins")) {
    r.kind = nn ? 1 : 2;
    int vb, ve;
    if (!header_value(s, n, vb, ve)) {
      r.err = T_HDR_COLON;
      return r;
    }
    const int q = py_int(s, vb, ve, &r.val);
    if (q == NUM_BAD) r.err = T_HDR_INT;
    if (q == NUM_RANGE) r.err = X_INT_RANGE;
    return r;
  }
  if (tok_eq(s, tb, te, "NetDegree")) {
    r.kind = 3;
    r.ne = -1;
    int vb, ve;
    if (!header_value(s, n, vb, ve)) {
      r.err = T_DEG_COLON;
      return r;
    }
    int p = vb, b0, e0;
    if (!next_tok(s, p, ve, b0, e0)) {
      r.err = T_DEG_INT;
      return r;
    }
    const int q = py_int(s, b0, e0, &r.val);
    if (q == NUM_BAD) r.err = T_DEG_INT;
    if (q == NUM_RANGE) r.err = X_INT_RANGE;
    if (q != NUM_OK) return r;
    int b1, e1;
    if (next_tok(s, p, ve, b1, e1)) {
      r.nb = b1;
      r.ne = e1;
    }
    return r;
  }
  r.kind = 4;
  r.nb = tb;
  r.ne = te;
  int b, e;
  while (next_tok(s, pos, n, b, e)) {
    if (tok_eq(s, b, e, ":")) {
      int b1, e1, b2, e2;
      if (next_tok(s, pos, n, b1, e1) && next_tok(s, pos, n, b2, e2)) {
        const int q1 = parse_float<HOST>(s, b1, e1, &r.dx);
        if (q1 == NUM_SLOW) {
          r.slow = 1;
          return r;
        }
        if (q1 == NUM_BAD) {
          r.err = T_OFFS;
          return r;
        }
        const int q2 = parse_float<HOST>(s, b2, e2, &r.dy);
        if (q2 == NUM_SLOW) {
          r.slow = 1;
          return r;
        }
        if (q2 == NUM_BAD) {
          r.err = T_OFFS;
          r.dx = 0.0;
        }
      }
      break;  // tokens.index(":") -- the first ':' token only
    }
  }
  return r;
}

template <bool HOST>
__host__ __device__ PlRec parse_pl_line(const char* s, int n) {  // netlist.py:313-327
  PlRec r{};
  int pos = 0, b1, e1, b2, e2;
  next_tok(s, pos, n, r.nb, r.ne);
  if (!next_tok(s, pos, n, b1, e1) || !next_tok(s, pos, n, b2, e2)) {
    r.err = P_FEW;
    return r;
  }
  const int q1 = parse_float<HOST>(s, b1, e1, &r.x);
  if (q1 == NUM_SLOW) {
    r.slow = 1;
    return r;
  }
  const int q2 = q1 == NUM_OK ? parse_float<HOST>(s, b2, e2, &r.y) : NUM_BAD;
  if (q2 == NUM_SLOW) {
    r.slow = 1;
    return r;
  }
  if (q1 == NUM_BAD || q2 == NUM_BAD) {
    r.err = P_NUM;
    return r;
  }
  int b, e;
  while (next_tok(s, pos, n, b, e))
    if (tok_eq(s, b, e, "/FIXED") || tok_eq(s, b, e, "/FIXED_NI")) r.fixed = 1;
  return r;
}

// ---- line splitting -------------------------------------------------------------
__global__ void k_line_heads(const char* __restrict__ t, int64_t len, uint8_t* __restrict__ head,
                             int* __restrict__ uni_ws) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const char p = i ? t[i - 1] : '\n';
    head[i] = (p == '\n' || (p == '\r' && t[i] != '\n')) ? 1 : 0;
    // Unicode whitespace (UTF-8) would split tokens in Python: not handled here
    const unsigned char c = (unsigned char)t[i];
    if (c == 0xC2 || c == 0xE1 || c == 0xE2 || c == 0xE3) {
      const unsigned char c1 = i + 1 < len ? (unsigned char)t[i + 1] : 0;
      const unsigned char c2 = i + 2 < len ? (unsigned char)t[i + 2] : 0;
      bool ws = false;
      if (c == 0xC2) ws = c1 == 0x85 || c1 == 0xA0;
      if (c == 0xE1) ws = c1 == 0x9A && c2 == 0x80;
      if (c == 0xE2) ws = (c1 == 0x80 && ((c2 >= 0x80 && c2 <= 0x8A) || c2 == 0xA8 || c2 == 0xA9 || c2 == 0xAF)) ||
                          (c1 == 0x81 && c2 == 0x9F);
      if (c == 0xE3) ws = c1 == 0x80 && c2 == 0x80;
      if (ws) atomicMin(uni_ws, (int)min(i, (int64_t)INT_MAX - 1));
    }
  }
}

// data line d: [beg, end) of the stripped text before '#'; keep = not blank, not "UCLA..."
__global__ void k_line_trim(const char* __restrict__ t, int64_t len, const int64_t* __restrict__ starts, int64_t nl,
                            int64_t* __restrict__ beg, int64_t* __restrict__ end, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = starts[i];
    const int64_t e0 = i + 1 < nl ? starts[i + 1] : len;
    int64_t e = b;
    while (e < e0 && t[e] != '#') ++e;
    while (b < e && is_ws((unsigned char)t[b])) ++b;
    while (e > b && is_ws((unsigned char)t[e - 1])) --e;
    beg[i] = b;
    end[i] = e;
    keep[i] = (e > b && !(e - b >= 4 && t[b] == 'U' && t[b + 1] == 'C' && t[b + 2] == 'L' && t[b + 3] == 'A')) ? 1 : 0;
  }
}

__global__ void k_gather_lines(int64_t nd, const int64_t* __restrict__ idx, const int64_t* __restrict__ beg,
                               const int64_t* __restrict__ end, int64_t* __restrict__ dbeg,
                               int64_t* __restrict__ dlen) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[d];
    dbeg[d] = beg[i];
    dlen[d] = end[i] - beg[i];
  }
}

// ---- names ------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t name_hash(const char* s, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ull ^ (uint64_t)n;
  for (int64_t i = 0; i < n; ++i) h = (h ^ (unsigned char)s[i]) * 0x100000001b3ull;
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h ? h : 1;  // 0 marks an empty table slot
}

__device__ __forceinline__ bool bytes_eq(const char* a, int64_t na, const char* b, int64_t nb) {
  if (na != nb) return false;
  for (int64_t i = 0; i < na; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

struct Names {  // cell names inside the .nodes text
  const char* text;
  const int64_t* beg;  // [ncells]
  const int32_t* len;
};

struct Table {
  uint64_t* keys;
  int32_t* vals;
  uint64_t mask;
};

__global__ void k_table_insert(int64_t n, const uint64_t* __restrict__ key_s, const int32_t* __restrict__ id_s,
                               Table tb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > 0 && key_s[i] == key_s[i - 1]) continue;  // duplicates were rejected before
    const uint64_t k = key_s[i];
    for (uint64_t s = k & tb.mask;; s = (s + 1) & tb.mask) {
      const unsigned long long old = atomicCAS((unsigned long long*)&tb.keys[s], 0ull, (unsigned long long)k);
      if (old == 0ull) {
        tb.vals[s] = id_s[i];
        break;
      }
    }
  }
}

__device__ __forceinline__ int32_t table_find(const Table& tb, const Names& nm, const char* s, int64_t n) {
  const uint64_t k = name_hash(s, n);
  for (uint64_t sl = k & tb.mask;; sl = (sl + 1) & tb.mask) {
    const uint64_t kk = tb.keys[sl];
    if (kk == 0) return -1;
    if (kk == k) {
      const int32_t id = tb.vals[sl];
      return bytes_eq(nm.text + nm.beg[id], nm.len[id], s, n) ? id : -1;
    }
  }
}

// ---- reductions helpers -------------------------------------------------------------
__device__ __forceinline__ unsigned long long ord_key(double v) {  // order-preserving map of doubles
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ inline double ord_val(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  memcpy(&v, &b, sizeof(v));
  return v;
}

// ---- .nodes ----------------------------------------------------------------------
__global__ void k_nodes_first_err(int64_t nd, const NodeRec* __restrict__ rec, unsigned long long* __restrict__ first) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    if (rec[d].err) atomicMin(first, (unsigned long long)d);
}

__global__ void k_nodes_cell_flag(int64_t nd, const NodeRec* __restrict__ rec, int64_t limit,
                                  uint8_t* __restrict__ flag) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    flag[d] = (d < limit && rec[d].kind == 0) ? 1 : 0;
}

__global__ void k_nodes_headers(int64_t nd, const NodeRec* __restrict__ rec, int64_t limit,
                                unsigned long long* __restrict__ last) {  // last[0] NumNodes, last[1] NumTerminals
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd && d < limit;
       d += (int64_t)gridDim.x * blockDim.x)
    if (rec[d].kind) atomicMax(&last[rec[d].kind - 1], (unsigned long long)d + 1);
}

__global__ void k_cells(int64_t nc, const int64_t* __restrict__ cell_line, const NodeRec* __restrict__ rec,
                        const int64_t* __restrict__ dbeg, const char* __restrict__ text, int64_t* __restrict__ nbeg,
                        int32_t* __restrict__ nlen, double* __restrict__ w, double* __restrict__ h,
                        uint8_t* __restrict__ term, uint64_t* __restrict__ key, int32_t* __restrict__ ids) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = cell_line[c];
    const NodeRec r = rec[d];
    nbeg[c] = dbeg[d] + r.nb;
    nlen[c] = r.ne - r.nb;
    w[c] = r.w;
    h[c] = r.h;
    term[c] = (uint8_t)r.term;
    key[c] = name_hash(text + nbeg[c], nlen[c]);
    ids[c] = (int32_t)c;
  }
}

// equal hashes: equal names are duplicates (the later cell is the error), different
// names a 64-bit collision (reported, never resolved silently)
__global__ void k_dups(int64_t nc, const uint64_t* __restrict__ key_s, const int32_t* __restrict__ id_s, Names nm,
                       unsigned long long* __restrict__ first_dup, int* __restrict__ collision) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    if (key_s[i] != key_s[i - 1]) continue;
    const int32_t a = id_s[i];
    bool dup = false;
    for (int64_t j = i - 1; j >= 0 && key_s[j] == key_s[i]; --j) {
      const int32_t b = id_s[j];
      if (bytes_eq(nm.text + nm.beg[a], nm.len[a], nm.text + nm.beg[b], nm.len[b])) {
        dup = true;
        break;
      }
    }
    if (dup)
      atomicMin(first_dup, (unsigned long long)a);
    else
      atomicExch(collision, 1);
  }
}

// ---- .nets -----------------------------------------------------------------------
__global__ void k_net_flags(int64_t nd, const NetRec* __restrict__ rec, int64_t* __restrict__ is_deg,
                            int64_t* __restrict__ is_pin) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x) {
    is_deg[d] = rec[d].kind == 3;
    is_pin[d] = rec[d].kind == 4;
  }
}

// deg_of[d] = nets started at or before d (inclusive scan), pin_rank[d] = pins before d
__global__ void k_deg_table(int64_t nd, const NetRec* __restrict__ rec, const int64_t* __restrict__ deg_of,
                            const int64_t* __restrict__ pin_rank, int64_t* __restrict__ deg_k,
                            int64_t* __restrict__ deg_pin0, int64_t* __restrict__ deg_line) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x) {
    if (rec[d].kind != 3) continue;
    const int64_t j = deg_of[d] - 1;
    deg_k[j] = rec[d].err ? 0 : rec[d].val;
    deg_pin0[j] = pin_rank[d];
    deg_line[j] = d;
  }
}

// pending of net j after its pins, or LLONG_MIN when a pin line overflowed it
// (that line is an error of its own, earlier)
__host__ __device__ __forceinline__ long long pending_after(long long k, long long pins) {
  if (k >= 0 && pins > k) return LLONG_MIN;
  return k - pins;
}

__global__ void k_net_errors(int64_t nd, const NetRec* __restrict__ rec, const int64_t* __restrict__ dbeg,
                             const char* __restrict__ text, const int64_t* __restrict__ deg_of,
                             const int64_t* __restrict__ pin_rank, const int64_t* __restrict__ deg_k,
                             const int64_t* __restrict__ deg_pin0, Table tb, Names nm, int32_t* __restrict__ pin_cell_line,
                             int* __restrict__ err, long long* __restrict__ err_val,
                             unsigned long long* __restrict__ first) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x) {
    const NetRec r = rec[d];
    int e = r.err;
    long long v = 0;
    if (r.kind == 3) {
      const int64_t j = deg_of[d] - 1;
      if (j > 0) {
        const long long p = pending_after(deg_k[j - 1], deg_pin0[j] - deg_pin0[j - 1]);
        if (p != 0 && p != LLONG_MIN) {
          e = T_PREV_MISSING;
          v = p;
        }
      }
    } else if (r.kind == 4) {
      const int64_t j = deg_of[d] - 1;
      bool outside = j < 0;
      if (!outside) {
        const long long k = deg_k[j];
        const long long pos = pin_rank[d] - deg_pin0[j] + 1;
        outside = k >= 0 && pos > k;
      }
      int32_t cell = -1;
      if (outside) {
        e = T_OUTSIDE;
      } else {
        cell = table_find(tb, nm, text + dbeg[d] + r.nb, r.ne - r.nb);
        if (cell < 0) e = T_DANGLING;
      }
      pin_cell_line[d] = cell;
    }
    err[d] = e;
    err_val[d] = v;
    if (e) atomicMin(first, (unsigned long long)d);
  }
}

__global__ void k_nets_headers(int64_t nd, const NetRec* __restrict__ rec, unsigned long long* __restrict__ last) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    if (rec[d].kind == 1) atomicMax(last, (unsigned long long)d + 1);
}

__global__ void k_pins_out(int64_t np, const int64_t* __restrict__ pin_line, const NetRec* __restrict__ rec,
                           const int32_t* __restrict__ pin_cell_line, int32_t* __restrict__ pin_cell,
                           double* __restrict__ dx, double* __restrict__ dy) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = pin_line[p];
    pin_cell[p] = pin_cell_line[d];
    dx[p] = rec[d].dx;
    dy[p] = rec[d].dy;
  }
}

__host__ __device__ __forceinline__ int dec_digits(int64_t v) {
  int k = 1;
  while (v >= 10) {
    v /= 10;
    ++k;
  }
  return k;
}

// net names: the NetDegree's second token, else f"net{j}" (netlist.py:280)
__global__ void k_net_name_len(int64_t nn, const int64_t* __restrict__ deg_line, const NetRec* __restrict__ rec,
                               int64_t* __restrict__ len) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn; j += (int64_t)gridDim.x * blockDim.x) {
    const NetRec r = rec[deg_line[j]];
    len[j] = r.ne >= 0 ? r.ne - r.nb : 3 + dec_digits(j);
  }
}

__global__ void k_net_name_fill(int64_t nn, const int64_t* __restrict__ deg_line, const NetRec* __restrict__ rec,
                                const int64_t* __restrict__ dbeg, const char* __restrict__ text,
                                const int64_t* __restrict__ off, char* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = deg_line[j];
    const NetRec r = rec[d];
    char* p = out + off[j];
    if (r.ne >= 0) {
      for (int i = r.nb; i < r.ne; ++i) *p++ = text[dbeg[d] + i];
    } else {
      p[0] = 'n'; p[1] = 'e'; p[2] = 't';
      const int k = dec_digits(j);
      int64_t v = j;
      for (int i = k - 1; i >= 0; --i) {
        p[3 + i] = (char)('0' + v % 10);
        v /= 10;
      }
    }
  }
}

struct IsPin {
  const NetRec* r;
  __host__ __device__ bool operator()(int64_t d) const { return r[d].kind == 4; }
};

// ---- .pl --------------------------------------------------------------------------
__global__ void k_pl_first_err(int64_t nd, const PlRec* __restrict__ rec, unsigned long long* __restrict__ first) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    if (rec[d].err) atomicMin(first, (unsigned long long)d);
}

__global__ void k_pl_assign(int64_t nd, const PlRec* __restrict__ rec, const int64_t* __restrict__ dbeg,
                            const char* __restrict__ text, Table tb, Names nm, unsigned long long* __restrict__ last,
                            unsigned long long* __restrict__ unknown) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x) {
    const PlRec r = rec[d];
    const int32_t c = table_find(tb, nm, text + dbeg[d] + r.nb, r.ne - r.nb);
    if (c < 0)
      atomicAdd(unknown, 1ull);
    else
      atomicMax(&last[c], (unsigned long long)d + 1);  // the dict keeps the last assignment
  }
}

__global__ void k_pl_cells(int64_t nc, const unsigned long long* __restrict__ last, const PlRec* __restrict__ rec,
                           const double* __restrict__ w, const double* __restrict__ h, uint8_t* __restrict__ fixed,
                           double* __restrict__ fixed_pos, unsigned long long* __restrict__ first_noplace,
                           unsigned long long* __restrict__ bbox, unsigned long long* __restrict__ n_placed) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long l = last[c];
    bool f = fixed[c] != 0;
    double fx = NAN, fy = NAN;
    if (l) {
      const PlRec r = rec[l - 1];
      f = f || r.fixed;
      if (f) {
        fx = __dadd_rn(r.x, __ddiv_rn(w[c], 2.0));  // netlist.py:437-438
        fy = __dadd_rn(r.y, __ddiv_rn(h[c], 2.0));
      }
      atomicMin(&bbox[0], ord_key(r.x));
      atomicMin(&bbox[1], ord_key(r.y));
      atomicMax(&bbox[2], ord_key(__dadd_rn(r.x, w[c])));
      atomicMax(&bbox[3], ord_key(__dadd_rn(r.y, h[c])));
      atomicAdd(n_placed, 1ull);
    } else if (f) {
      atomicMin(first_noplace, (unsigned long long)c);
    }
    fixed[c] = f ? 1 : 0;
    fixed_pos[2 * c] = fx;
    fixed_pos[2 * c + 1] = fy;
  }
}

}  // namespace bs

// ---- the parse driver ----------------------------------------------------------------

namespace {

using namespace bs;

template <typename T>
T* own(Ctx* ctx, Bookshelf* B, int64_t count) {
  void* p = dev_alloc(ctx, (size_t)std::max<int64_t>(count, 1) * sizeof(T) + 16);
  B->owned.push_back(p);
  return static_cast<T*>(p);
}

template <typename T>
T fetch1(Ctx* ctx, const T* d) {
  T h;
  GIFT_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void flagged_positions(Ctx* ctx, const uint8_t* flags, int64_t n, int64_t* out, int64_t* d_count) {
  thrust::counting_iterator<int64_t> it(0);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_count, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flags, out, d_count, n, ctx->stream));
  ctx->launches += 1;
}

void scan_excl(Ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, ctx->stream));
  ctx->launches += 1;
}

void scan_incl(Ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, in, out, n, ctx->stream));
  ctx->launches += 1;
}

// a parse error: "<file>\t<lineno>\t<code>\t<value>\t<payload>" for the Python shim
[[noreturn]] void parse_error(int file, int64_t lineno, int code, long long value, const std::string& payload) {
  throw_error(GIFT_ERR_PARSE, std::to_string(file) + "\t" + std::to_string(lineno) + "\t" + std::to_string(code) +
                                  "\t" + std::to_string(value) + "\t" + payload);
}

// device copy of a file + its data lines
struct Lines {
  DevBuf<char> text;
  DevBuf<int64_t> beg, len, line;  // per data line: start, length, index of the physical line (0-based)
  int64_t nd = 0;
};

void split_lines(Ctx* ctx, int file, const char* h, int64_t n, Lines& L) {
  cudaStream_t st = ctx->stream;
  L.text = DevBuf<char>(ctx, n + 1);
  if (n == 0) return;
  GIFT_CUDA(cudaMemcpyAsync(L.text.p, h, n, cudaMemcpyHostToDevice, st));
  DevBuf<uint8_t> head(ctx, n);
  DevBuf<int> uni(ctx, 1);
  const int big = INT_MAX;
  GIFT_CUDA(cudaMemcpyAsync(uni.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_line_heads<<<grid_for(n, kBlock), kBlock, 0, st>>>(L.text.p, n, head.p, uni.p);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<int64_t> starts(ctx, n), cnt(ctx, 2);
  flagged_positions(ctx, head.p, n, starts.p, cnt.p);
  const int64_t nl = fetch1(ctx, cnt.p);
  const int uws = fetch1(ctx, uni.p);
  if (uws != INT_MAX)
    throw_error(GIFT_ERR_VALUE, "file " + std::to_string(file) + " byte " + std::to_string(uws) +
                                    ": non-ASCII whitespace is not supported by the device Bookshelf reader");
  head.reset();
  DevBuf<int64_t> b(ctx, nl), e(ctx, nl);
  DevBuf<uint8_t> keep(ctx, nl);
  k_line_trim<<<grid_for(nl, kBlock), kBlock, 0, st>>>(L.text.p, n, starts.p, nl, b.p, e.p, keep.p);
  GIFT_LAUNCH_CHECK(ctx);
  L.line = DevBuf<int64_t>(ctx, nl);
  flagged_positions(ctx, keep.p, nl, L.line.p, cnt.p);
  L.nd = fetch1(ctx, cnt.p);
  L.beg = DevBuf<int64_t>(ctx, L.nd);
  L.len = DevBuf<int64_t>(ctx, L.nd);
  if (L.nd) {
    k_gather_lines<<<grid_for(L.nd, kBlock), kBlock, 0, st>>>(L.nd, L.line.p, b.p, e.p, L.beg.p, L.len.p);
    GIFT_LAUNCH_CHECK(ctx);
  }
}

std::string host_line(Ctx* ctx, const char* h, const Lines& L, int64_t d) {
  int64_t b = 0, n = 0;
  GIFT_CUDA(cudaMemcpyAsync(&b, L.beg.p + d, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaMemcpyAsync(&n, L.len.p + d, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return std::string(h + b, (size_t)n);
}

int64_t lineno_of(Ctx* ctx, const Lines& L, int64_t d) { return fetch1(ctx, L.line.p + d) + 1; }

template <class Rec>
__global__ void k_slow_flags(int64_t nd, const Rec* __restrict__ rec, uint8_t* __restrict__ flag) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    flag[d] = rec[d].slow ? 1 : 0;
}

template <class Rec>
__global__ void k_slow_gather(int64_t ns, const int64_t* __restrict__ idx, const int64_t* __restrict__ beg,
                              const int64_t* __restrict__ len, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    out[2 * i] = beg[idx[i]];
    out[2 * i + 1] = len[idx[i]];
  }
}

template <class Rec>
__global__ void k_slow_scatter(int64_t ns, const int64_t* __restrict__ idx, const Rec* __restrict__ fixed,
                               Rec* __restrict__ rec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
    rec[idx[i]] = fixed[i];
}

// lines the device left undecided (rare number spellings): re-parse just those
// on the host from the caller's buffer with the same line parser + strtod
template <class Rec, Rec (*HostParse)(const char*, int)>
void resolve_slow(Ctx* ctx, const char* h, const Lines& L, Rec* rec) {
  if (L.nd == 0) return;
  cudaStream_t st = ctx->stream;
  DevBuf<uint8_t> flag(ctx, L.nd);
  DevBuf<int64_t> idx(ctx, L.nd), cnt(ctx, 2);
  k_slow_flags<Rec><<<grid_for(L.nd, kBlock), kBlock, 0, st>>>(L.nd, rec, flag.p);
  GIFT_LAUNCH_CHECK(ctx);
  flagged_positions(ctx, flag.p, L.nd, idx.p, cnt.p);
  const int64_t ns = fetch1(ctx, cnt.p);
  if (ns == 0) return;
  DevBuf<int64_t> bl(ctx, 2 * ns);
  k_slow_gather<Rec><<<grid_for(ns, kBlock), kBlock, 0, st>>>(ns, idx.p, L.beg.p, L.len.p, bl.p);
  GIFT_LAUNCH_CHECK(ctx);
  std::vector<int64_t> hbl(2 * ns);
  GIFT_CUDA(cudaMemcpyAsync(hbl.data(), bl.p, 2 * ns * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  std::vector<Rec> hr(ns);
  for (int64_t i = 0; i < ns; ++i) hr[i] = HostParse(h + hbl[2 * i], (int)hbl[2 * i + 1]);
  DevBuf<Rec> fixed(ctx, ns);
  GIFT_CUDA(cudaMemcpyAsync(fixed.p, hr.data(), ns * sizeof(Rec), cudaMemcpyHostToDevice, st));
  k_slow_scatter<Rec><<<grid_for(ns, kBlock), kBlock, 0, st>>>(ns, idx.p, fixed.p, rec);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaStreamSynchronize(st));
}

NodeRec node_dev(const char* s, int n) { return parse_node_line<true>(s, n); }
NetRec net_dev(const char* s, int n) { return parse_net_line<true>(s, n); }
PlRec pl_dev(const char* s, int n) { return parse_pl_line<true>(s, n); }

__device__ NodeRec node_parse_d(const char* s, int n) { return parse_node_line<false>(s, n); }
__device__ NetRec net_parse_d(const char* s, int n) { return parse_net_line<false>(s, n); }
__device__ PlRec pl_parse_d(const char* s, int n) { return parse_pl_line<false>(s, n); }

template <class Rec, Rec (*Parse)(const char*, int)>
__global__ void k_parse_lines(const char* __restrict__ t, int64_t nd, const int64_t* __restrict__ beg,
                              const int64_t* __restrict__ len, Rec* __restrict__ rec) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    rec[d] = Parse(t + beg[d], (int)len[d]);
}

}  // namespace

Bookshelf* bookshelf_parse(Ctx* ctx, const char* h_nodes, int64_t n_nodes, const char* h_nets, int64_t n_nets,
                           const char* h_pl, int64_t n_pl) {
  cudaStream_t st = ctx->stream;
  std::unique_ptr<Bookshelf> B(new Bookshelf());
  auto fail_cleanup = [&]() {
    for (void* p : B->owned) dev_free(ctx, p);
    B->owned.clear();
  };
  try {
    const unsigned long long NONE = ULLONG_MAX;
    // ======================= .nodes (file 0) =======================
    Lines LN;
    split_lines(ctx, 0, h_nodes, n_nodes, LN);
    DevBuf<NodeRec> nrec(ctx, LN.nd);
    if (LN.nd) {
      k_parse_lines<NodeRec, node_parse_d><<<grid_for(LN.nd, kBlock), kBlock, 0, st>>>(LN.text.p, LN.nd, LN.beg.p,
                                                                                     LN.len.p, nrec.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    resolve_slow<NodeRec, node_dev>(ctx, h_nodes, LN, nrec.p);
    DevBuf<unsigned long long> red(ctx, 8);
    GIFT_CUDA(cudaMemsetAsync(red.p, 0xff, 8 * sizeof(unsigned long long), st));
    if (LN.nd) {
      k_nodes_first_err<<<grid_for(LN.nd, kBlock), kBlock, 0, st>>>(LN.nd, nrec.p, red.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    const unsigned long long first_local = fetch1(ctx, red.p);
    const int64_t limit = first_local == NONE ? LN.nd : (int64_t)first_local;
    DevBuf<uint8_t> cflag(ctx, LN.nd);
    DevBuf<int64_t> cell_line(ctx, LN.nd), cnt(ctx, 2);
    int64_t nc = 0;
    if (LN.nd) {
      k_nodes_cell_flag<<<grid_for(LN.nd, kBlock), kBlock, 0, st>>>(LN.nd, nrec.p, limit, cflag.p);
      GIFT_LAUNCH_CHECK(ctx);
      flagged_positions(ctx, cflag.p, LN.nd, cell_line.p, cnt.p);
      nc = fetch1(ctx, cnt.p);
    }
    if (nc >= INT_MAX) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^31 - 1 cells");
    int64_t* nbeg = own<int64_t>(ctx, B.get(), nc);
    int32_t* nlen = own<int32_t>(ctx, B.get(), nc);
    B->width = own<double>(ctx, B.get(), nc);
    B->height = own<double>(ctx, B.get(), nc);
    B->fixed = own<uint8_t>(ctx, B.get(), nc);
    DevBuf<uint64_t> key(ctx, nc), key_s(ctx, nc);
    DevBuf<int32_t> ids(ctx, nc), id_s(ctx, nc);
    if (nc) {
      k_cells<<<grid_for(nc, kBlock), kBlock, 0, st>>>(nc, cell_line.p, nrec.p, LN.beg.p, LN.text.p, nbeg, nlen,
                                                       B->width, B->height, B->fixed, key.p, ids.p);
      GIFT_LAUNCH_CHECK(ctx);
      size_t bytes = 0;
      GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key_s.p, ids.p, id_s.p, nc, 0, 64, st));
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key_s.p, ids.p, id_s.p, nc, 0, 64, st));
      ctx->launches += 1;
    }
    Names nm{LN.text.p, nbeg, nlen};
    DevBuf<int> coll(ctx, 1);
    GIFT_CUDA(cudaMemsetAsync(coll.p, 0, sizeof(int), st));
    if (nc > 1) {
      k_dups<<<grid_for(nc, kBlock), kBlock, 0, st>>>(nc, key_s.p, id_s.p, nm, red.p + 1, coll.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    const unsigned long long first_dup_cell = fetch1(ctx, red.p + 1);
    if (fetch1(ctx, coll.p)) throw_error(GIFT_ERR_INTERNAL, "64-bit cell-name hash collision");
    {
      // the first error in line order: a local one, or the first duplicate
      int64_t d_err = -1;
      int code = 0;
      if (first_dup_cell != NONE) {
        d_err = fetch1(ctx, cell_line.p + first_dup_cell);
        code = N_DUP;
      }
      if (first_local != NONE && (d_err < 0 || (int64_t)first_local < d_err)) {
        d_err = (int64_t)first_local;
        code = fetch1(ctx, nrec.p + d_err).err;
      }
      if (d_err >= 0) {
        const NodeRec r = fetch1(ctx, nrec.p + d_err);
        const std::string line = host_line(ctx, h_nodes, LN, d_err);
        parse_error(0, lineno_of(ctx, LN, d_err), code, 0,
                    code == N_DUP ? line.substr(r.nb, r.ne - r.nb) : line);
      }
    }
    // headers: the last NumNodes / NumTerminals line wins
    GIFT_CUDA(cudaMemsetAsync(red.p + 2, 0, 2 * sizeof(unsigned long long), st));
    if (LN.nd) {
      k_nodes_headers<<<grid_for(LN.nd, kBlock), kBlock, 0, st>>>(LN.nd, nrec.p, LN.nd, red.p + 2);
      GIFT_LAUNCH_CHECK(ctx);
    }
    const unsigned long long hn = fetch1(ctx, red.p + 2), ht = fetch1(ctx, red.p + 3);
    if (hn) {
      const long long num_nodes = fetch1(ctx, nrec.p + (hn - 1)).hval;
      if (num_nodes != nc) parse_error(0, 0, N_COUNT, num_nodes, std::to_string(nc));
    }
    B->n_terminals_decl = ht ? fetch1(ctx, nrec.p + (ht - 1)).hval : -1;
    B->n_cells = nc;
    // names table (capacity >= 2 x cells, power of two)
    uint64_t cap = 1024;
    while (cap < 2 * (uint64_t)nc) cap <<= 1;
    DevBuf<uint64_t> tkeys(ctx, cap);
    DevBuf<int32_t> tvals(ctx, cap);
    GIFT_CUDA(cudaMemsetAsync(tkeys.p, 0, cap * sizeof(uint64_t), st));
    Table tb{tkeys.p, tvals.p, cap - 1};
    if (nc) {
      k_table_insert<<<grid_for(nc, kBlock), kBlock, 0, st>>>(nc, key_s.p, id_s.p, tb);
      GIFT_LAUNCH_CHECK(ctx);
    }
    key.reset();
    key_s.reset();
    ids.reset();
    id_s.reset();
    nrec.reset();
    // ======================= .nets (file 1) =======================
    Lines LT;
    split_lines(ctx, 1, h_nets, n_nets, LT);
    const int64_t nd = LT.nd;
    DevBuf<NetRec> trec(ctx, nd);
    if (nd) {
      k_parse_lines<NetRec, net_parse_d><<<grid_for(nd, kBlock), kBlock, 0, st>>>(LT.text.p, nd, LT.beg.p, LT.len.p,
                                                                                trec.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    resolve_slow<NetRec, net_dev>(ctx, h_nets, LT, trec.p);
    DevBuf<int64_t> is_deg(ctx, nd + 1), is_pin(ctx, nd + 1), deg_of(ctx, nd + 1), pin_rank(ctx, nd + 1);
    int64_t ndeg = 0, npin = 0;
    if (nd) {
      k_net_flags<<<grid_for(nd, kBlock), kBlock, 0, st>>>(nd, trec.p, is_deg.p, is_pin.p);
      GIFT_LAUNCH_CHECK(ctx);
      GIFT_CUDA(cudaMemsetAsync(is_pin.p + nd, 0, sizeof(int64_t), st));
      scan_incl(ctx, is_deg.p, deg_of.p, nd);
      scan_excl(ctx, is_pin.p, pin_rank.p, nd + 1);
      ndeg = fetch1(ctx, deg_of.p + nd - 1);
      npin = fetch1(ctx, pin_rank.p + nd);
    }
    DevBuf<int64_t> deg_k(ctx, ndeg + 1), deg_pin0(ctx, ndeg + 1), deg_line(ctx, ndeg + 1);
    DevBuf<int32_t> pin_cell_line(ctx, nd);
    DevBuf<int> terr(ctx, nd);
    DevBuf<long long> terr_val(ctx, nd);
    if (nd) {
      k_deg_table<<<grid_for(nd, kBlock), kBlock, 0, st>>>(nd, trec.p, deg_of.p, pin_rank.p, deg_k.p, deg_pin0.p,
                                                           deg_line.p);
      GIFT_LAUNCH_CHECK(ctx);
      GIFT_CUDA(cudaMemcpyAsync(deg_pin0.p + ndeg, &npin, sizeof(int64_t), cudaMemcpyHostToDevice, st));
      k_net_errors<<<grid_for(nd, kBlock), kBlock, 0, st>>>(nd, trec.p, LT.beg.p, LT.text.p, deg_of.p, pin_rank.p,
                                                            deg_k.p, deg_pin0.p, tb, nm, pin_cell_line.p, terr.p,
                                                            terr_val.p, red.p + 4);
      GIFT_LAUNCH_CHECK(ctx);
      const unsigned long long fe = fetch1(ctx, red.p + 4);
      if (fe != NONE) {
        const int code = fetch1(ctx, terr.p + fe);
        const NetRec r = fetch1(ctx, trec.p + fe);
        const std::string line = host_line(ctx, h_nets, LT, (int64_t)fe);
        parse_error(1, lineno_of(ctx, LT, (int64_t)fe), code, fetch1(ctx, terr_val.p + fe),
                    code == T_DANGLING ? line.substr(r.nb, r.ne - r.nb) : line);
      }
    }
    if (ndeg) {  // the last net's pending pin lines (netlist.py:306-307)
      const long long k = fetch1(ctx, deg_k.p + ndeg - 1);
      const long long p = pending_after(k, npin - fetch1(ctx, deg_pin0.p + ndeg - 1));
      if (p != 0) parse_error(1, 0, T_LAST_MISSING, p, "");
    }
    {
      GIFT_CUDA(cudaMemsetAsync(red.p + 5, 0, sizeof(unsigned long long), st));
      if (nd) {
        k_nets_headers<<<grid_for(nd, kBlock), kBlock, 0, st>>>(nd, trec.p, red.p + 5);
        GIFT_LAUNCH_CHECK(ctx);
      }
      const unsigned long long hl = fetch1(ctx, red.p + 5);
      if (hl) {
        const long long num_nets = fetch1(ctx, trec.p + (hl - 1)).val;
        if (num_nets != ndeg) parse_error(1, 0, T_COUNT, num_nets, std::to_string(ndeg));
      }
    }
    B->n_nets = ndeg;
    B->n_pins = npin;
    B->net_start = own<int64_t>(ctx, B.get(), ndeg + 1);
    GIFT_CUDA(cudaMemcpyAsync(B->net_start, deg_pin0.p, (ndeg + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    B->pin_cell = own<int32_t>(ctx, B.get(), npin);
    B->pin_dx = own<double>(ctx, B.get(), npin);
    B->pin_dy = own<double>(ctx, B.get(), npin);
    if (npin) {
      DevBuf<int64_t> pin_line(ctx, npin);
      thrust::counting_iterator<int64_t> it(0);
      size_t bytes = 0;
      GIFT_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, pin_line.p, cnt.p, nd, IsPin{trec.p}, st));
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceSelect::If(tmp.p, bytes, it, pin_line.p, cnt.p, nd, IsPin{trec.p}, st));
      ctx->launches += 1;
      k_pins_out<<<grid_for(npin, kBlock), kBlock, 0, st>>>(npin, pin_line.p, trec.p, pin_cell_line.p, B->pin_cell,
                                                            B->pin_dx, B->pin_dy);
      GIFT_LAUNCH_CHECK(ctx);
    }
    // net names
    B->net_name_off = own<int64_t>(ctx, B.get(), ndeg + 1);
    if (ndeg) {
      DevBuf<int64_t> nl(ctx, ndeg + 1);
      GIFT_CUDA(cudaMemsetAsync(nl.p + ndeg, 0, sizeof(int64_t), st));
      k_net_name_len<<<grid_for(ndeg, kBlock), kBlock, 0, st>>>(ndeg, deg_line.p, trec.p, nl.p);
      GIFT_LAUNCH_CHECK(ctx);
      scan_excl(ctx, nl.p, B->net_name_off, ndeg + 1);
      B->net_name_bytes = fetch1(ctx, B->net_name_off + ndeg);
      B->net_names = own<char>(ctx, B.get(), B->net_name_bytes);
      k_net_name_fill<<<grid_for(ndeg, kBlock), kBlock, 0, st>>>(ndeg, deg_line.p, trec.p, LT.beg.p, LT.text.p,
                                                                 B->net_name_off, B->net_names);
      GIFT_LAUNCH_CHECK(ctx);
    } else {
      GIFT_CUDA(cudaMemsetAsync(B->net_name_off, 0, sizeof(int64_t), st));
      B->net_names = own<char>(ctx, B.get(), 0);
    }
    trec.reset();
    // ======================= .pl (file 2) =======================
    Lines LP;
    split_lines(ctx, 2, h_pl, n_pl, LP);
    DevBuf<PlRec> prec(ctx, LP.nd);
    if (LP.nd) {
      k_parse_lines<PlRec, pl_parse_d><<<grid_for(LP.nd, kBlock), kBlock, 0, st>>>(LP.text.p, LP.nd, LP.beg.p,
                                                                                 LP.len.p, prec.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    resolve_slow<PlRec, pl_dev>(ctx, h_pl, LP, prec.p);
    if (LP.nd) {
      k_pl_first_err<<<grid_for(LP.nd, kBlock), kBlock, 0, st>>>(LP.nd, prec.p, red.p + 6);
      GIFT_LAUNCH_CHECK(ctx);
      const unsigned long long fe = fetch1(ctx, red.p + 6);
      if (fe != NONE) {
        const int code = fetch1(ctx, prec.p + fe).err;
        parse_error(2, lineno_of(ctx, LP, (int64_t)fe), code, 0, host_line(ctx, h_pl, LP, (int64_t)fe));
      }
    }
    DevBuf<unsigned long long> last(ctx, nc), acc(ctx, 8);
    GIFT_CUDA(cudaMemsetAsync(last.p, 0, std::max<int64_t>(nc, 1) * sizeof(unsigned long long), st));
    const unsigned long long init[8] = {ULLONG_MAX, ULLONG_MAX, 0, 0, 0, 0, ULLONG_MAX, 0};
    GIFT_CUDA(cudaMemcpyAsync(acc.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    if (LP.nd) {
      k_pl_assign<<<grid_for(LP.nd, kBlock), kBlock, 0, st>>>(LP.nd, prec.p, LP.beg.p, LP.text.p, tb, nm, last.p,
                                                              acc.p + 4);
      GIFT_LAUNCH_CHECK(ctx);
    }
    B->fixed_pos = own<double>(ctx, B.get(), 2 * nc);
    if (nc) {
      k_pl_cells<<<grid_for(nc, kBlock), kBlock, 0, st>>>(nc, last.p, prec.p, B->width, B->height, B->fixed,
                                                          B->fixed_pos, acc.p + 6, acc.p, acc.p + 5);
      GIFT_LAUNCH_CHECK(ctx);
    }
    unsigned long long ha[8];
    GIFT_CUDA(cudaMemcpyAsync(ha, acc.p, sizeof(ha), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    B->pl_unknown = (int64_t)ha[4];
    B->n_placed = (int64_t)ha[5];
    for (int i = 0; i < 4; ++i) B->bbox[i] = ord_val(ha[i]);
    // cell names (bytes + offsets), before the .nodes text goes away
    B->cell_name_off = own<int64_t>(ctx, B.get(), nc + 1);
    {
      std::vector<int64_t> hb(nc);
      std::vector<int32_t> hl(nc);
      GIFT_CUDA(cudaMemcpyAsync(hb.data(), nbeg, nc * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      GIFT_CUDA(cudaMemcpyAsync(hl.data(), nlen, nc * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      GIFT_CUDA(cudaStreamSynchronize(st));
      std::vector<int64_t> off(nc + 1, 0);
      for (int64_t c = 0; c < nc; ++c) off[c + 1] = off[c] + hl[c];
      B->cell_name_bytes = off[nc];
      std::string names;
      names.reserve((size_t)off[nc]);
      for (int64_t c = 0; c < nc; ++c) names.append(h_nodes + hb[c], (size_t)hl[c]);
      B->cell_names = own<char>(ctx, B.get(), off[nc]);
      GIFT_CUDA(cudaMemcpyAsync(B->cell_name_off, off.data(), (nc + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      if (off[nc])
        GIFT_CUDA(cudaMemcpyAsync(B->cell_names, names.data(), off[nc], cudaMemcpyHostToDevice, st));
      GIFT_CUDA(cudaStreamSynchronize(st));
    }
    if (ha[6] != ULLONG_MAX) {  // a fixed cell without a placement (netlist.py:440-442)
      std::vector<char> nmv;
      int64_t o[2];
      GIFT_CUDA(cudaMemcpy(o, B->cell_name_off + ha[6], 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
      nmv.resize(o[1] - o[0]);
      if (!nmv.empty()) GIFT_CUDA(cudaMemcpy(nmv.data(), B->cell_names + o[0], nmv.size(), cudaMemcpyDeviceToHost));
      parse_error(2, 0, P_NOPLACE, 0, std::string(nmv.begin(), nmv.end()));
    }
    {
      std::vector<uint8_t> hf(nc);
      GIFT_CUDA(cudaMemcpyAsync(hf.data(), B->fixed, nc, cudaMemcpyDeviceToHost, st));
      GIFT_CUDA(cudaStreamSynchronize(st));
      int64_t k = 0;
      for (uint8_t v : hf) k += v;
      B->n_fixed = k;
    }
    return B.release();
  } catch (...) {
    fail_cleanup();
    throw;
  }
}

void bookshelf_destroy(Ctx* ctx, Bookshelf* B) {
  if (!B) return;
  for (void* p : B->owned) dev_free(ctx, p);
  delete B;
}

}  // namespace gift
