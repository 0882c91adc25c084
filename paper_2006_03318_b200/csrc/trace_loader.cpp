// trace_loader.cpp -- native columnar reader/writer of kernsim trace documents.
//
// Replaces kernsim.trace.parse_trace (pkg/src/kernsim/trace.py:281-328) for
// large traces: the JSON document is read straight into the columns the
// device ingest consumes (ks_ingest / ks_map_layers), with the reference's
// validation (trace.py:147-252) and its error precedence:
//
//   JSON syntax (MalformedDocument) > top-level type > schema_version >
//   time_unit > events type > first bad event (document order) > duplicate
//   id > lane overlap (check_lane_overlaps, trace.py:255-265) > layer_markers
//   type > first bad marker > marker overlap (trace.py:268-278).
//
// gradient_buckets and metadata are small; their byte spans are returned and
// the Python host validates them (trace.py:231-252, 317-326) after this.
//
// Times: us_to_ns (trace.py:92-98) is Decimal(str(value)) * 1000 rounded
// half-up.  str() of a JSON float is Python's shortest round-trip repr, so a
// float literal is converted to that decimal first: literals with <= 15
// significant digits are their own shortest repr (DBL_DIG), others go through
// strtod + std::to_chars (shortest).  Half-up rounding of a decimal is "first
// dropped digit >= 5 rounds away from zero", done on the digit string.
//
// Parallelism: one pre-scan pass over the text (per chunk: unescaped-quote
// parity, bracket depth under both string-state hypotheses, first '{' per
// relative depth) gives, after a prefix over chunks, exact split points at
// element boundaries of the events / layer_markers arrays; threads parse the
// elements of their slice into local columns, which are merged (lane / name
// interning in document order) into the handle.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <memory>
#include <string>
#include <string_view>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "ddsim.h"
#include "host_alloc.h"

namespace ddsim {
void set_last_error(const std::string& msg);  // graph.cu
}
using ddsim::set_last_error;

namespace {

enum VT : uint8_t { V_ABSENT = 0, V_NULL, V_TRUE, V_FALSE, V_INT, V_FLOAT, V_STR, V_ARR, V_OBJ };

struct Val {
  VT t = V_ABSENT;
  bool esc = false;       // string contains backslash escapes
  const char* p = nullptr;  // token span (strings: content without quotes)
  int64_t n = 0;
};

constexpr int kKinds = 7;
const char* const kKindNames[kKinds] = {"CpuApi", "CpuOther", "GpuKernel", "GpuMemcpy",
                                        "DataLoad", "Comm", "Sync"};
// KIND_CODE (trace.py host mirror): 0 CpuApi 1 CpuOther 2 GpuKernel 3 GpuMemcpy
// 4 DataLoad 5 Comm 6 Sync.  CPU_KINDS = {0,1,4,6}, GPU_KINDS = {2,3}.
inline bool kind_is_cpu(int k) { return k == 0 || k == 1 || k == 4 || k == 6; }
inline bool kind_is_gpu(int k) { return k == 2 || k == 3; }
const char* const kPhaseNames[3] = {"Forward", "Backward", "WeightUpdate"};

// error classes, in the order the reference would raise them
enum ErrCode { E_NONE = 0, E_MALFORMED = KS_ERR_MALFORMED, E_SCHEMA = KS_ERR_SCHEMA,
               E_OVERLAP = KS_ERR_OVERLAP, E_UNSUPPORTED = KS_ERR_UNSUPPORTED };

struct Err {
  int code = E_NONE;
  std::string msg;
  void set(int c, std::string m) {
    if (code == E_NONE) { code = c; msg = std::move(m); }
  }
};

// ------------------------------------------------------------------ lexer

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

// bytes that end a plain run inside a JSON string: quote, backslash, controls
struct StrSpecial {
  bool t[256] = {};
  StrSpecial() {
    for (int c = 0; c < 0x20; ++c) t[c] = true;
    t[(unsigned char)'"'] = true;
    t[(unsigned char)'\\'] = true;
  }
};
const StrSpecial kStrSpecial;

struct Lexer {
  const char* s;
  const char* e;
  const char* cur;
  bool bad = false;
  const char* badpos = nullptr;

  Lexer(const char* b, const char* end, const char* at) : s(b), e(end), cur(at) {}

  void fail() {
    if (!bad) { bad = true; badpos = cur; }
  }
  inline void ws() {
    while (cur < e && is_ws(*cur)) ++cur;
  }
  inline int peek() const { return cur < e ? (unsigned char)*cur : -1; }

  static int hexv(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
  }

  bool string(Val& v) {  // at '"'
    ++cur;
    const char* b = cur;
    bool esc = false;
    for (;;) {
      while (cur < e && !kStrSpecial.t[(unsigned char)*cur]) ++cur;  // plain bytes
      if (cur >= e) { fail(); return false; }
      unsigned char c = (unsigned char)*cur;
      if (c == '"') break;
      if (c < 0x20) { fail(); return false; }  // json strict mode
      if (c == '\\') {
        esc = true;
        ++cur;
        if (cur >= e) { fail(); return false; }
        char x = *cur;
        if (x == 'u') {
          if (e - cur < 5) { fail(); return false; }
          for (int k = 1; k <= 4; ++k)
            if (hexv(cur[k]) < 0) { fail(); return false; }
          cur += 5;
          continue;
        }
        if (!(x == '"' || x == '\\' || x == '/' || x == 'b' || x == 'f' || x == 'n' ||
              x == 'r' || x == 't')) { fail(); return false; }
        ++cur;
        continue;
      }
      ++cur;
    }
    v.t = V_STR;
    v.p = b;
    v.n = cur - b;
    v.esc = esc;
    ++cur;
    return true;
  }

  bool number(Val& v) {
    const char* b = cur;
    bool flt = false;
    if (cur < e && *cur == '-') ++cur;
    if (cur >= e) { fail(); return false; }
    if (*cur == '0') {
      ++cur;
    } else if (*cur >= '1' && *cur <= '9') {
      while (cur < e && *cur >= '0' && *cur <= '9') ++cur;
    } else {
      fail();
      return false;
    }
    if (cur < e && *cur == '.') {
      const char* d = cur + 1;
      if (d < e && *d >= '0' && *d <= '9') {
        cur = d;
        while (cur < e && *cur >= '0' && *cur <= '9') ++cur;
        flt = true;
      }  // else: "1." -> python json stops before '.', then "Extra data"
    }
    if (cur < e && (*cur == 'e' || *cur == 'E')) {
      const char* d = cur + 1;
      if (d < e && (*d == '+' || *d == '-')) ++d;
      if (d < e && *d >= '0' && *d <= '9') {
        cur = d;
        while (cur < e && *cur >= '0' && *cur <= '9') ++cur;
        flt = true;
      }
    }
    v.t = flt ? V_FLOAT : V_INT;
    v.p = b;
    v.n = cur - b;
    return true;
  }

  bool lit(const char* w, int n) {
    if (e - cur >= n && std::memcmp(cur, w, n) == 0) { cur += n; return true; }
    return false;
  }

  // any value; containers are validated and skipped (span recorded)
  bool value(Val& v, int depth = 0) {
    ws();
    int c = peek();
    switch (c) {
      case '"': return string(v);
      case '{': case '[': {
        const char* b = cur;
        if (!skip_container(depth)) return false;
        v.t = (c == '{') ? V_OBJ : V_ARR;
        v.p = b;
        v.n = cur - b;
        return true;
      }
      case 't': if (lit("true", 4)) { v.t = V_TRUE; return true; } break;
      case 'f': if (lit("false", 5)) { v.t = V_FALSE; return true; } break;
      case 'n': if (lit("null", 4)) { v.t = V_NULL; return true; } break;
      case 'N': if (lit("NaN", 3)) { v.t = V_FLOAT; v.p = cur - 3; v.n = 3; return true; } break;
      case 'I':
        if (lit("Infinity", 8)) { v.t = V_FLOAT; v.p = cur - 8; v.n = 8; return true; }
        break;
      default:
        if (c == '-' && e - cur >= 9 && std::memcmp(cur, "-Infinity", 9) == 0) {
          cur += 9; v.t = V_FLOAT; v.p = cur - 9; v.n = 9; return true;
        }
        if (c == '-' || (c >= '0' && c <= '9')) return number(v);
    }
    fail();
    return false;
  }

  bool skip_container(int depth) {
    if (depth > 100000) { fail(); return false; }
    char open = *cur++;
    char close = open == '{' ? '}' : ']';
    ws();
    if (peek() == close) { ++cur; return true; }
    for (;;) {
      Val tmp;
      if (open == '{') {
        ws();
        if (peek() != '"' || !string(tmp)) { fail(); return false; }
        ws();
        if (peek() != ':') { fail(); return false; }
        ++cur;
      }
      if (!value(tmp, depth + 1)) return false;
      ws();
      int c = peek();
      if (c == ',') { ++cur; ws(); continue; }
      if (c == close) { ++cur; return true; }
      fail();
      return false;
    }
  }
};

// ------------------------------------------------------------ conversions

void put_utf8(std::string& o, uint32_t cp) {
  if (cp < 0x80) {
    o += char(cp);
  } else if (cp < 0x800) {
    o += char(0xC0 | (cp >> 6));
    o += char(0x80 | (cp & 0x3F));
  } else if (cp < 0x10000) {
    o += char(0xE0 | (cp >> 12));
    o += char(0x80 | ((cp >> 6) & 0x3F));
    o += char(0x80 | (cp & 0x3F));
  } else {
    o += char(0xF0 | (cp >> 18));
    o += char(0x80 | ((cp >> 12) & 0x3F));
    o += char(0x80 | ((cp >> 6) & 0x3F));
    o += char(0x80 | (cp & 0x3F));
  }
}

std::string unescape(const Val& v) {
  if (!v.esc) return std::string(v.p, (size_t)v.n);
  std::string o;
  o.reserve((size_t)v.n);
  const char* c = v.p;
  const char* e = v.p + v.n;
  while (c < e) {
    if (*c != '\\') { o += *c++; continue; }
    ++c;
    char x = *c++;
    switch (x) {
      case 'b': o += '\b'; break;
      case 'f': o += '\f'; break;
      case 'n': o += '\n'; break;
      case 'r': o += '\r'; break;
      case 't': o += '\t'; break;
      case 'u': {
        uint32_t cp = 0;
        for (int k = 0; k < 4; ++k) cp = cp * 16 + Lexer::hexv(c[k]);
        c += 4;
        if (cp >= 0xD800 && cp < 0xDC00 && e - c >= 6 && c[0] == '\\' && c[1] == 'u') {
          uint32_t lo = 0;
          bool ok = true;
          for (int k = 0; k < 4; ++k) {
            int h = Lexer::hexv(c[2 + k]);
            if (h < 0) ok = false;
            lo = lo * 16 + (h < 0 ? 0 : h);
          }
          if (ok && lo >= 0xDC00 && lo < 0xE000) {
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            c += 6;
          }
        }
        put_utf8(o, cp);  // lone surrogates kept as 3-byte sequences
        break;
      }
      default: o += x;  // '"' '\\' '/'
    }
  }
  return o;
}

bool str_eq(const Val& v, const char* w) {
  if (v.t != V_STR) return false;
  size_t n = std::strlen(w);
  if (!v.esc) return (size_t)v.n == n && std::memcmp(v.p, w, n) == 0;
  return unescape(v) == w;
}

// A decimal number: value = (neg ? -1 : 1) * digits * 10^exp, digits without
// leading zeros ("" = 0).
struct Dec {
  bool neg = false;
  std::string digits;
  int64_t exp = 0;
};

// digits/exponent of a JSON number literal (exact decimal value of the text)
void literal_dec(const char* p, int64_t n, Dec& d) {
  const char* e = p + n;
  d = Dec();
  if (p < e && *p == '-') { d.neg = true; ++p; }
  int64_t frac = 0;
  bool in_frac = false;
  for (; p < e && *p != 'e' && *p != 'E'; ++p) {
    if (*p == '.') { in_frac = true; continue; }
    if (!(d.digits.empty() && *p == '0')) d.digits += *p;
    if (in_frac) ++frac;
  }
  int64_t x = 0;
  if (p < e) {  // exponent
    ++p;
    bool xn = false;
    if (*p == '+' || *p == '-') xn = (*p++ == '-');
    for (; p < e; ++p) x = std::min<int64_t>(x * 10 + (*p - '0'), (int64_t)1 << 40);
    if (xn) x = -x;
  }
  d.exp = x - frac;
  while (!d.digits.empty() && d.digits.back() == '0') { d.digits.pop_back(); ++d.exp; }
}

// decimal of Python's str(float(literal)); false for non-finite values
bool float_repr_dec(const Val& v, Dec& d) {
  if (v.n >= 3 && (v.p[v.n - 1] == 'N' || v.p[v.n - 1] == 'y')) return false;  // NaN/Infinity
  literal_dec(v.p, v.n, d);
  if (d.digits.empty()) return true;  // 0.0 / -0.0 -> Decimal('0.0') / '-0.0' == 0
  int64_t adj = d.exp + (int64_t)d.digits.size() - 1;  // decimal exponent of the leading digit
  if (d.digits.size() <= 15 && adj > -290 && adj < 290) return true;  // own shortest repr
  std::string lit(v.p, (size_t)v.n);
  double x = std::strtod(lit.c_str(), nullptr);
  if (!std::isfinite(x)) return false;
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  literal_dec(buf, r.ptr - buf, d);
  return true;
}

// Decimal(str) of a JSON string: ASCII decimal with optional surrounding
// whitespace and digit-grouping underscores.  0 ok, 1 invalid (Decimal
// raises -> SchemaViolation), 2 unsupported (non-ASCII / inf / nan).
int string_dec(const Val& v, Dec& d) {
  std::string s = unescape(v);
  for (unsigned char c : s)
    if (c >= 0x80) return 2;
  size_t b = 0, e = s.size();
  auto sp = [](char c) { return c == ' ' || (c >= '\t' && c <= '\r'); };
  while (b < e && sp(s[b])) ++b;
  while (e > b && sp(s[e - 1])) --e;
  std::string t = s.substr(b, e - b);
  std::string low;
  for (char c : t) low += (char)std::tolower((unsigned char)c);
  std::string body = (!low.empty() && (low[0] == '+' || low[0] == '-')) ? low.substr(1) : low;
  if (body == "inf" || body == "infinity" || body == "nan" || body == "snan" ||
      (body.size() > 3 && (body.rfind("nan", 0) == 0 || body.rfind("snan", 0) == 0)))
    return 2;
  // decimal strips whitespace and drops every '_' (Decimal('1__0') == 10), then
  // sign? (digits [. digits?] | . digits) ([eE] sign? digits)?
  std::string u;
  for (char c : t)
    if (c != '_') u += c;
  t.swap(u);
  size_t i = 0;
  std::string lit;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) { if (t[i] == '-') lit += '-'; ++i; }
  auto digits = [&](std::string& out) {
    size_t st = i;
    while (i < t.size() && t[i] >= '0' && t[i] <= '9') out += t[i++];
    return i > st;
  };
  std::string ip, fp, xp;
  bool hi = digits(ip);
  bool hf = false;
  if (i < t.size() && t[i] == '.') { ++i; hf = digits(fp); }
  if (!hi && !hf) return 1;
  lit += ip.empty() ? "0" : ip;
  if (!fp.empty()) lit += "." + fp;
  if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
    ++i;
    std::string sg;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) sg = t[i++];
    if (!digits(xp)) return 1;
    lit += "e" + sg + xp;
  }
  if (i != t.size()) return 1;
  literal_dec(lit.data(), (int64_t)lit.size(), d);
  return 0;
}

// round_half_up(d * 1000) into int64; false on overflow
bool dec_to_ns(const Dec& d, int64_t& out) {
  if (d.digits.empty()) { out = 0; return true; }
  int64_t k = d.exp + 3;
  int64_t len = (int64_t)d.digits.size();
  unsigned __int128 mag = 0;
  const unsigned __int128 lim = (unsigned __int128)INT64_MAX;
  if (k >= 0) {
    if (len + k > 19) return false;
    for (char c : d.digits) mag = mag * 10 + (c - '0');
    for (int64_t j = 0; j < k; ++j) mag *= 10;
  } else {
    int64_t keep = len + k;  // digits left of the point
    if (keep > 19) return false;
    for (int64_t j = 0; j < keep; ++j) mag = mag * 10 + (d.digits[(size_t)j] - '0');
    char first = keep >= 0 ? d.digits[(size_t)keep] : '0';
    if (first >= '5') mag += 1;
  }
  if (mag > lim) return false;
  out = d.neg ? -(int64_t)mag : (int64_t)mag;
  return true;
}

// us_to_ns of any JSON value: 0 ok, 1 SchemaViolation, 2 unsupported
int value_to_ns(const Val& v, int64_t& out) {
  if (v.t == V_INT || v.t == V_FLOAT) {
    // fast path: "-?I(.F)?" with <= 15 digits is its own shortest repr
    const char* p = v.p;
    const char* e = v.p + v.n;
    bool neg = false;
    if (*p == '-') { neg = true; ++p; }
    const char* ib = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    const char* ie = p;
    const char* fb = p;
    const char* fe = p;
    if (p < e && *p == '.') {
      fb = ++p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
      fe = p;
    }
    if (p == e && (ie - ib) + (fe - fb) <= 15) {
      int64_t m = 0;
      for (const char* q = ib; q < ie; ++q) m = m * 10 + (*q - '0');
      for (int k = 0; k < 3; ++k) m = m * 10 + (fb + k < fe ? fb[k] - '0' : 0);
      if (fb + 3 < fe && fb[3] >= '5') ++m;
      out = neg ? -m : m;
      return 0;
    }
  }
  Dec d;
  switch (v.t) {
    case V_INT: literal_dec(v.p, v.n, d); break;
    case V_FLOAT:
      if (!float_repr_dec(v, d)) return 2;
      break;
    case V_STR: {
      int r = string_dec(v, d);
      if (r) return r;
      break;
    }
    default: return 1;  // Decimal('True'/'None'/'[..]') raises
  }
  return dec_to_ns(d, out) ? 0 : 2;
}

// isinstance(x, int) (bool included) and x >= 0: 0 ok, 1 not, 2 too large
int value_to_nonneg_int(const Val& v, int64_t& out) {
  if (v.t == V_TRUE) { out = 1; return 0; }
  if (v.t == V_FALSE) { out = 0; return 0; }
  if (v.t != V_INT) return 1;
  if (v.p[0] != '-' && v.n <= 18) {
    int64_t x = 0;
    for (int64_t j = 0; j < v.n; ++j) x = x * 10 + (v.p[j] - '0');
    out = x;
    return 0;
  }
  Dec d;
  literal_dec(v.p, v.n, d);
  if (d.digits.empty()) { out = 0; return 0; }
  if (d.neg) return 1;
  if ((int64_t)d.digits.size() + d.exp > 18) return 2;
  int64_t x = 0;
  for (char c : d.digits) x = x * 10 + (c - '0');
  for (int64_t j = 0; j < d.exp; ++j) x *= 10;
  out = x;
  return 0;
}

// str(value) for names / layers: 0 ok, 2 unsupported (floats, containers)
int value_to_str(const Val& v, std::string& out) {
  switch (v.t) {
    case V_STR: out = unescape(v); return 0;
    case V_TRUE: out = "True"; return 0;
    case V_FALSE: out = "False"; return 0;
    case V_NULL: out = "None"; return 0;
    case V_INT: {
      Dec d;
      literal_dec(v.p, v.n, d);
      if (d.digits.empty()) { out = "0"; return 0; }
      out = std::string(v.p, (size_t)v.n);  // JSON ints have no leading zeros
      return 0;
    }
    default: return 2;
  }
}

// LaneId.parse (trace.py:56-62): "<cpu|gpu|comm>:<key>", key non-empty.
// returns class code (0 cpu, 1 gpu, 2 comm) or -1
int lane_class_of(std::string_view s) {
  size_t c = s.find(':');
  if (c == std::string_view::npos || c + 1 >= s.size()) return -1;
  std::string_view p(s.data(), c);
  if (p == "cpu") return 0;
  if (p == "gpu") return 1;
  if (p == "comm") return 2;
  return -1;
}

std::string py_repr_str(std::string_view s) {  // enough of repr() for messages
  std::string o = "'";
  for (char c : s) {
    if (c == '\'' || c == '\\') o += '\\';
    o += c;
  }
  return o + "'";
}

std::string val_repr(const Val& v) {
  switch (v.t) {
    case V_STR: return py_repr_str(unescape(v));
    case V_NULL: case V_ABSENT: return "None";
    case V_TRUE: return "True";
    case V_FALSE: return "False";
    default: return std::string(v.p, (size_t)std::min<int64_t>(v.n, 64));
  }
}

// --------------------------------------------------------- interning

// string -> dense id in first-appearance order (open addressing, lookups by view)
struct Interner {
  std::vector<std::string> items;
  std::vector<uint64_t> hashes;
  std::vector<int32_t> slots = std::vector<int32_t>(64, -1);

  static uint64_t hash(std::string_view s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h ^ (h >> 29);
  }
  int32_t get(std::string_view s) {
    uint64_t h = hash(s);
    size_t mask = slots.size() - 1;
    size_t i = (size_t)h & mask;
    while (slots[i] >= 0) {
      int32_t k = slots[i];
      if (hashes[(size_t)k] == h && items[(size_t)k] == s) return k;
      i = (i + 1) & mask;
    }
    int32_t k = (int32_t)items.size();
    items.emplace_back(s);
    hashes.push_back(h);
    slots[i] = k;
    if (items.size() * 2 > slots.size()) {  // grow
      std::vector<int32_t> ns(slots.size() * 2, -1);
      size_t m2 = ns.size() - 1;
      for (size_t j = 0; j < items.size(); ++j) {
        size_t q = (size_t)hashes[j] & m2;
        while (ns[q] >= 0) q = (q + 1) & m2;
        ns[q] = (int32_t)j;
      }
      slots.swap(ns);
    }
    return k;
  }
};

// view of a string value (unescaped into `scratch` only when it has escapes)
inline std::string_view sv_of(const Val& v, std::string& scratch) {
  if (!v.esc) return std::string_view(v.p, (size_t)v.n);
  scratch = unescape(v);
  return scratch;
}

// ------------------------------------------------------- object parsing

// Parse one object's members; `slot(key) -> Val*` (nullptr = ignore).
template <class SlotFn>
bool parse_object(Lexer& L, SlotFn slot) {
  // at '{'
  ++L.cur;
  L.ws();
  if (L.peek() == '}') { ++L.cur; return true; }
  for (;;) {
    L.ws();
    Val k;
    if (L.peek() != '"' || !L.string(k)) { L.fail(); return false; }
    L.ws();
    if (L.peek() != ':') { L.fail(); return false; }
    ++L.cur;
    Val v;
    if (!L.value(v)) return false;
    Val* dst = slot(k);
    if (dst) *dst = v;
    L.ws();
    int c = L.peek();
    if (c == ',') { ++L.cur; continue; }
    if (c == '}') { ++L.cur; return true; }
    L.fail();
    return false;
  }
}

inline bool key_is(const Val& k, const char* w, size_t n) {
  if (!k.esc) return (size_t)k.n == n && std::memcmp(k.p, w, n) == 0;
  return unescape(k) == std::string(w, n);
}

// messages of LaneId.parse / us_to_ns carry no "events[i]: " context
const std::string kNoCtx = "\x01";

std::string with_ctx(const std::string& where, const std::string& m) {
  if (!m.empty() && m[0] == '\x01') return m.substr(1);
  return where + m;
}

// --------------------------------------------------------- event sink

struct EventChunk {
  hvec<int64_t> id, start, dur, corr, size;
  hvec<uint8_t> kind, dtoh;
  hvec<int32_t> lane, sync, name;
  Interner lanes, names;
  std::vector<int64_t> lane_first_ev, lane_first_sync;  // per local lane, local row (or -1)
  Err err;
  int64_t err_row = -1;

  int32_t lane_ix(std::string_view s, int64_t row, bool as_sync) {
    int32_t k = lanes.get(s);
    if ((size_t)k == lane_first_ev.size()) {
      lane_first_ev.push_back(-1);
      lane_first_sync.push_back(-1);
    }
    auto& f = as_sync ? lane_first_sync[(size_t)k] : lane_first_ev[(size_t)k];
    if (f < 0) f = row;
    return k;
  }
  size_t rows() const { return id.size(); }
  void reserve(size_t k) {
    id.reserve(k); start.reserve(k); dur.reserve(k); corr.reserve(k); size.reserve(k);
    kind.reserve(k); dtoh.reserve(k); lane.reserve(k); sync.reserve(k); name.reserve(k);
  }
};

struct EvFields {
  Val kind, id, lane, start, duration, correlation, size_bytes, sync_target, name;
};

// _event_from (trace.py:147-199) on one parsed element; appends a row or
// records the first error of this chunk.  `index` is the global position
// (only for messages; the chunk's offset is patched in later).
void event_element(Lexer& L, EventChunk& ch, int64_t local_index) {
  EvFields f;
  if (L.peek() != '{') {
    Val v;
    if (!L.value(v)) return;
    if (ch.err.code == E_NONE) {
      ch.err.set(E_SCHEMA, ": not an object");
      ch.err_row = local_index;
    }
    return;
  }
  bool ok = parse_object(L, [&](const Val& k) -> Val* {
    switch (k.esc ? 'x' : (k.n ? k.p[0] : 0)) {
      case 'k': if (key_is(k, "kind", 4)) return &f.kind; break;
      case 'i': if (key_is(k, "id", 2)) return &f.id; break;
      case 'l': if (key_is(k, "lane", 4)) return &f.lane; break;
      case 's':
        if (key_is(k, "start", 5)) return &f.start;
        if (key_is(k, "size_bytes", 10)) return &f.size_bytes;
        if (key_is(k, "sync_target", 11)) return &f.sync_target;
        break;
      case 'd': if (key_is(k, "duration", 8)) return &f.duration; break;
      case 'c': if (key_is(k, "correlation", 11)) return &f.correlation; break;
      case 'n': if (key_is(k, "name", 4)) return &f.name; break;
      case 'x': {
        std::string u = unescape(k);
        if (u == "kind") return &f.kind;
        if (u == "id") return &f.id;
        if (u == "lane") return &f.lane;
        if (u == "start") return &f.start;
        if (u == "duration") return &f.duration;
        if (u == "correlation") return &f.correlation;
        if (u == "size_bytes") return &f.size_bytes;
        if (u == "sync_target") return &f.sync_target;
        if (u == "name") return &f.name;
        break;
      }
    }
    return nullptr;
  });
  if (!ok || ch.err.code != E_NONE) return;  // after the first error: syntax only
  auto fail = [&](int code, std::string m) {
    ch.err.set(code, (!m.empty() && m[0] == '\x01') ? m : ": " + m);
    ch.err_row = local_index;
  };
  if (f.kind.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'kind'");
  int kind = -1;
  std::string s_kind, s_lane, s_target, s_name;
  if (f.kind.t == V_STR) {
    std::string_view ks = sv_of(f.kind, s_kind);
    for (int j = 0; j < kKinds; ++j)
      if (ks == kKindNames[j]) { kind = j; break; }
  }
  if (kind < 0) return fail(E_SCHEMA, "unknown kind " + val_repr(f.kind));
  if (f.id.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'id'");
  int64_t id = 0;
  int r = value_to_nonneg_int(f.id, id);
  if (r == 1) return fail(E_SCHEMA, "id must be a non-negative integer");
  if (r == 2) return fail(E_UNSUPPORTED, "id does not fit in int64");
  if (f.lane.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'lane'");
  if (f.lane.t != V_STR) return fail(E_SCHEMA, kNoCtx + "invalid lane id " + val_repr(f.lane));
  std::string_view lane = sv_of(f.lane, s_lane);
  int lc = lane_class_of(lane);
  if (lc < 0) return fail(E_SCHEMA, kNoCtx + "invalid lane id " + py_repr_str(lane));
  if (f.start.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'start'");
  int64_t start = 0, dur = 0;
  r = value_to_ns(f.start, start);
  if (r) return fail(r == 1 ? E_SCHEMA : E_UNSUPPORTED, kNoCtx + "bad time value " + val_repr(f.start));
  if (f.duration.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'duration'");
  r = value_to_ns(f.duration, dur);
  if (r) return fail(r == 1 ? E_SCHEMA : E_UNSUPPORTED, kNoCtx + "bad time value " + val_repr(f.duration));
  if (start < 0 || dur < 0) return fail(E_SCHEMA, "negative start or duration");
  int64_t corr = -1, size = -1;
  if (f.correlation.t != V_ABSENT && f.correlation.t != V_NULL) {
    r = value_to_nonneg_int(f.correlation, corr);
    if (r == 1) return fail(E_SCHEMA, "correlation must be a non-negative integer");
    if (r == 2) return fail(E_UNSUPPORTED, "correlation does not fit in int64");
  }
  if (f.size_bytes.t != V_ABSENT && f.size_bytes.t != V_NULL) {
    r = value_to_nonneg_int(f.size_bytes, size);
    if (r == 1) return fail(E_SCHEMA, "size_bytes must be a non-negative integer");
    if (r == 2) return fail(E_UNSUPPORTED, "size_bytes does not fit in int64");
  }
  bool has_target = f.sync_target.t != V_ABSENT && f.sync_target.t != V_NULL;
  std::string_view target;
  if (has_target) {
    if (f.sync_target.t != V_STR)
      return fail(E_SCHEMA, kNoCtx + "invalid lane id " + val_repr(f.sync_target));
    target = sv_of(f.sync_target, s_target);
    if (lane_class_of(target) < 0) return fail(E_SCHEMA, kNoCtx + "invalid lane id " + py_repr_str(target));
  }
  if (kind_is_gpu(kind) && corr < 0)
    return fail(E_SCHEMA, std::string(kKindNames[kind]) + " events require a correlation id");
  if (kind_is_gpu(kind) && lc != 1)
    return fail(E_SCHEMA, std::string(kKindNames[kind]) + " events must be on a gpu lane");
  if (kind_is_cpu(kind) && lc != 0)
    return fail(E_SCHEMA, std::string(kKindNames[kind]) + " events must be on a cpu lane");
  if (kind == 5 && lc != 2) return fail(E_SCHEMA, "Comm events must be on a comm lane");
  if (has_target && kind != 6) return fail(E_SCHEMA, "sync_target only allowed on Sync events");
  if (f.name.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'name'");
  std::string_view name;
  if (f.name.t == V_STR) {
    name = sv_of(f.name, s_name);
  } else {
    if (value_to_str(f.name, s_name)) return fail(E_UNSUPPORTED, "non-scalar or float name");
    name = s_name;
  }

  int64_t row = (int64_t)ch.rows();
  ch.id.push_back(id);
  ch.kind.push_back((uint8_t)kind);
  ch.lane.push_back(ch.lane_ix(lane, row, false));
  ch.start.push_back(start);
  ch.dur.push_back(dur);
  ch.corr.push_back(corr);
  ch.size.push_back(size);
  ch.sync.push_back(has_target ? ch.lane_ix(target, row, true) : -1);
  ch.dtoh.push_back(name.size() >= 11 && name.compare(0, 11, "memcpy_dtoh") == 0);
  ch.name.push_back(ch.names.get(name));
}

// --------------------------------------------------------- marker sink

struct MarkerChunk {
  std::vector<int64_t> start, end;
  std::vector<int32_t> lane, layer;
  std::vector<uint8_t> phase;
  Interner lanes, layers;
  Err err;
  int64_t err_row = -1;
  size_t rows() const { return start.size(); }
  void reserve(size_t k) {
    start.reserve(k); end.reserve(k); lane.reserve(k); layer.reserve(k); phase.reserve(k);
  }
};

void marker_element(Lexer& L, MarkerChunk& ch, int64_t local_index) {
  struct { Val layer, phase, cpu_lane, start, end; } f;
  if (L.peek() != '{') {
    Val v;
    if (!L.value(v)) return;
    if (ch.err.code == E_NONE) {
      ch.err.set(E_SCHEMA, ": not an object");
      ch.err_row = local_index;
    }
    return;
  }
  bool ok = parse_object(L, [&](const Val& k) -> Val* {
    std::string u = k.esc ? unescape(k) : std::string(k.p, (size_t)k.n);
    if (u == "layer") return &f.layer;
    if (u == "phase") return &f.phase;
    if (u == "cpu_lane") return &f.cpu_lane;
    if (u == "start") return &f.start;
    if (u == "end") return &f.end;
    return nullptr;
  });
  if (!ok || ch.err.code != E_NONE) return;
  auto fail = [&](int code, std::string m) {
    ch.err.set(code, (!m.empty() && m[0] == '\x01') ? m : ": " + m);
    ch.err_row = local_index;
  };
  if (f.phase.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'phase'");
  int phase = -1;
  if (f.phase.t == V_STR) {
    std::string ps = unescape(f.phase);
    for (int j = 0; j < 3; ++j)
      if (ps == kPhaseNames[j]) phase = j;
  }
  if (phase < 0) return fail(E_SCHEMA, "unknown phase " + val_repr(f.phase));
  if (f.cpu_lane.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'cpu_lane'");
  if (f.cpu_lane.t != V_STR) return fail(E_SCHEMA, kNoCtx + "invalid lane id " + val_repr(f.cpu_lane));
  std::string lane = unescape(f.cpu_lane);
  int lc = lane_class_of(lane);
  if (lc < 0) return fail(E_SCHEMA, kNoCtx + "invalid lane id " + py_repr_str(lane));
  if (lc != 0) return fail(E_SCHEMA, "cpu_lane must be a cpu lane");
  int64_t st = 0, en = 0;
  if (f.start.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'start'");
  int r = value_to_ns(f.start, st);
  if (r) return fail(r == 1 ? E_SCHEMA : E_UNSUPPORTED, kNoCtx + "bad time value " + val_repr(f.start));
  if (f.end.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'end'");
  r = value_to_ns(f.end, en);
  if (r) return fail(r == 1 ? E_SCHEMA : E_UNSUPPORTED, kNoCtx + "bad time value " + val_repr(f.end));
  if (!(st < en)) return fail(E_SCHEMA, "start must be < end");
  if (f.layer.t == V_ABSENT) return fail(E_SCHEMA, "missing field 'layer'");
  std::string layer;
  if (value_to_str(f.layer, layer)) return fail(E_UNSUPPORTED, "non-scalar or float layer");
  ch.start.push_back(st);
  ch.end.push_back(en);
  ch.lane.push_back(ch.lanes.get(lane));
  ch.layer.push_back(ch.layers.get(layer));
  ch.phase.push_back((uint8_t)phase);
}

// ------------------------------------------------------ parallel arrays

struct PreScan {
  // per chunk
  std::vector<int64_t> begin;
  std::vector<uint8_t> parity;   // unescaped quotes mod 2
  std::vector<uint8_t> bs_out;   // chunk ends inside an odd backslash run
  std::vector<int64_t> dA, dB;   // depth delta, start outside (A) / inside (B) a string
  // after prefix
  std::vector<uint8_t> in_str;
  std::vector<int64_t> depth;
  std::vector<int64_t> first2;   // first '{' at absolute depth 2 (array elements), -1 none
};

inline uint64_t prefix_xor(uint64_t x) {
  x ^= x << 1; x ^= x << 2; x ^= x << 4; x ^= x << 8; x ^= x << 16; x ^= x << 32;
  return x;
}

// 64-byte block -> bitmasks of backslash, quote, open ({[), close (}]) bytes
struct Masks { uint64_t bs, q, op, cl; };

inline Masks block_masks(const uint8_t* p) {
  Masks m{0, 0, 0, 0};
#if defined(__SSE2__)
  const __m128i vbs = _mm_set1_epi8('\\'), vq = _mm_set1_epi8('"');
  const __m128i vob = _mm_set1_epi8('{'), vos = _mm_set1_epi8('[');
  const __m128i vcb = _mm_set1_epi8('}'), vcs = _mm_set1_epi8(']');
  for (int k = 0; k < 4; ++k) {
    __m128i x = _mm_loadu_si128((const __m128i*)(p + 16 * k));
    uint64_t sh = 16 * k;
    m.bs |= (uint64_t)(uint32_t)_mm_movemask_epi8(_mm_cmpeq_epi8(x, vbs)) << sh;
    m.q |= (uint64_t)(uint32_t)_mm_movemask_epi8(_mm_cmpeq_epi8(x, vq)) << sh;
    m.op |= (uint64_t)(uint32_t)_mm_movemask_epi8(
        _mm_or_si128(_mm_cmpeq_epi8(x, vob), _mm_cmpeq_epi8(x, vos))) << sh;
    m.cl |= (uint64_t)(uint32_t)_mm_movemask_epi8(
        _mm_or_si128(_mm_cmpeq_epi8(x, vcb), _mm_cmpeq_epi8(x, vcs))) << sh;
  }
#else
  for (int i = 0; i < 64; ++i) {
    uint8_t c = p[i];
    m.bs |= (uint64_t)(c == '\\') << i;
    m.q |= (uint64_t)(c == '"') << i;
    m.op |= (uint64_t)(c == '{' || c == '[') << i;
    m.cl |= (uint64_t)(c == '}' || c == ']') << i;
  }
#endif
  return m;
}

// bits of characters escaped by an odd backslash run (carry = run entering the block)
inline uint64_t escaped_bits(uint64_t bs, uint32_t& carry) {
  if (!bs && !carry) return 0;
  uint64_t esc = 0;
  uint32_t c = carry;
  for (int i = 0; i < 64; ++i) {
    uint32_t b = (bs >> i) & 1;
    esc |= (uint64_t)(c & (b ^ 1) ? 1 : 0) << i;  // non-backslash after odd run
    esc |= (uint64_t)(c & b) << i;                 // escaped backslash
    c = b & (c ^ 1);
  }
  carry = c;
  return esc;
}

// pass 1 over chunk k: quote parity and depth deltas under both hypotheses
void prescan_chunk(const char* s, int64_t b, int64_t e, PreScan& ps, size_t k) {
  uint32_t bs = 0;  // entering inside an odd backslash run?
  for (int64_t j = b - 1; j >= 0 && s[j] == '\\'; --j) bs ^= 1;
  uint64_t instr = 0;  // hypothesis A (outside at b): 1 = inside a string
  int64_t dA = 0, dB = 0;
  uint32_t par = 0;
  const uint8_t* u = (const uint8_t*)s;
  int64_t i = b;
  uint8_t tail[64];
  while (i < e) {
    const uint8_t* p = u + i;
    int64_t len = std::min<int64_t>(64, e - i);
    if (len < 64) {
      std::memset(tail, ' ', 64);
      std::memcpy(tail, p, (size_t)len);
      p = tail;
    }
    Masks m = block_masks(p);
    uint64_t esc = escaped_bits(m.bs, bs);
    uint64_t q = m.q & ~esc;
    uint64_t x = prefix_xor(q) ^ instr;  // 1 = inside a string (hypothesis A)
    instr = (uint64_t)0 - (x >> 63);
    par ^= (uint32_t)__builtin_popcountll(q) & 1;
    uint64_t op = m.op, cl = m.cl;
    dA += __builtin_popcountll(op & ~x) - __builtin_popcountll(cl & ~x);
    dB += __builtin_popcountll(op & x) - __builtin_popcountll(cl & x);
    i += len;
  }
  ps.parity[k] = (uint8_t)par;
  ps.bs_out[k] = (uint8_t)bs;
  ps.dA[k] = dA;
  ps.dB[k] = dB;
}

// pass 2: from a chunk start with known state, the first '{' at depth 2
int64_t first_elem_brace(const char* s, int64_t b, int64_t e, bool in_str, int64_t depth) {
  bool bs = false;
  for (int64_t j = b - 1; j >= 0 && s[j] == '\\'; --j) bs = !bs;
  for (int64_t i = b; i < e; ++i) {
    char c = s[i];
    if (in_str) {
      if (bs) { bs = false; continue; }
      if (c == '\\') { bs = true; continue; }
      if (c == '"') in_str = false;
      continue;
    }
    if (c == '"') { in_str = true; continue; }
    if (c == '{' || c == '[') {
      if (c == '{' && depth == 2) return i;
      ++depth;
    } else if (c == '}' || c == ']') {
      --depth;
    }
  }
  return -1;
}

// K work items on T threads (atomic work counter; items are independent)
template <class F>
void pool_for(size_t K, int T, F fn) {
  const int W = (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(T, 1), K));
  if (W == 1) {
    for (size_t k = 0; k < K; ++k) fn(k);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (int w = 0; w < W; ++w)
    th.emplace_back([&] {
      for (size_t k; (k = next.fetch_add(1)) < K;) fn(k);
    });
  for (auto& t : th) t.join();
}

// K pre-scan chunks (fine-grained, so arrays much smaller than n / T still
// get many split points) on T threads.
PreScan prescan(const char* s, int64_t n, int K0, int T) {
  auto tp0 = std::chrono::steady_clock::now();
  PreScan ps;
  int64_t step = ((n + K0 - 1) / K0 + 63) / 64 * 64;
  size_t K = (size_t)K0;
  ps.begin.resize(K + 1);
  for (size_t k = 0; k <= K; ++k) ps.begin[k] = std::min<int64_t>((int64_t)k * step, n);
  ps.parity.assign(K, 0);
  ps.bs_out.assign(K, 0);
  ps.dA.assign(K, 0);
  ps.dB.assign(K, 0);
  pool_for(K, T, [&](size_t k) { prescan_chunk(s, ps.begin[k], ps.begin[k + 1], ps, k); });
  if (std::getenv("DDSIM_TRACE_TIMING"))
    std::fprintf(stderr, "[prescan] pass1 %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count());
  ps.in_str.assign(K + 1, 0);
  ps.depth.assign(K + 1, 0);
  for (size_t k = 0; k < K; ++k) {
    ps.in_str[k + 1] = ps.in_str[k] ^ ps.parity[k];
    ps.depth[k + 1] = ps.depth[k] + (ps.in_str[k] ? ps.dB[k] : ps.dA[k]);
  }
  auto tq0 = std::chrono::steady_clock::now();
  ps.first2.assign(K, -1);
  pool_for(K, T, [&](size_t k) {
    ps.first2[k] = first_elem_brace(s, ps.begin[k], ps.begin[k + 1], ps.in_str[k], ps.depth[k]);
  });
  if (std::getenv("DDSIM_TRACE_TIMING"))
    std::fprintf(stderr, "[prescan] pass2 %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tq0).count());
  return ps;
}

// Split points of the array whose '[' is at `open` (elements at depth 2):
// the first element '{' of every prescan chunk after `open`.
std::vector<int64_t> split_points(const PreScan& ps, int64_t open) {
  std::vector<int64_t> sp;
  for (size_t k = 0; k < ps.first2.size(); ++k) {
    int64_t pos = ps.first2[k];
    if (ps.begin[k] > open && pos > open && (sp.empty() || pos > sp.back())) sp.push_back(pos);
  }
  return sp;
}

struct SliceResult {
  int64_t end = -1;      // position after ']' if this slice closed the array
  bool reached_next = false;
  bool syntax = false;
  int64_t syntax_pos = -1;
  int64_t count = 0;     // elements parsed
};

// Parse array elements from `from` (first: just after '[') until the cursor
// lands on `stop` after a comma, or the closing ']'.
template <class Chunk, class Elem>
SliceResult parse_slice(const char* s, int64_t n, int64_t from, int64_t stop, bool first,
                        Chunk& ch, Elem elem) {
  SliceResult r;
  Lexer L(s, s + n, s + from);
  ch.reserve((size_t)(((stop >= 0 ? stop : n) - from) / 64 + 16));  // virtual only until touched
  if (first) {
    L.ws();
    if (L.peek() == ']') { r.end = (L.cur - s) + 1; return r; }
  }
  for (;;) {
    L.ws();
    if (stop >= 0 && (L.cur - s) >= stop) {
      r.reached_next = (L.cur - s) == stop;
      if (!r.reached_next) L.fail();
      break;
    }
    elem(L, ch, r.count);
    if (L.bad) break;
    ++r.count;
    L.ws();
    int c = L.peek();
    if (c == ',') {
      ++L.cur;
      continue;
    }
    if (c == ']') { r.end = (L.cur - s) + 1; return r; }
    L.fail();
    break;
  }
  if (L.bad) { r.syntax = true; r.syntax_pos = L.badpos - s; }
  return r;
}

template <class Chunk, class Elem>
struct ArrayParse {
  std::vector<Chunk> chunks;
  std::vector<int64_t> first_index;  // global element index of each chunk's first element
  int64_t end = -1;
  bool syntax = false;
  int64_t syntax_pos = -1;
};

template <class Chunk, class Elem>
ArrayParse<Chunk, Elem> parse_array(const char* s, int64_t n, int64_t open,
                                    const std::vector<int64_t>& sp, Elem elem, int T) {
  ArrayParse<Chunk, Elem> ap;
  size_t K = sp.size() + 1;
  ap.chunks.resize(K);
  std::vector<SliceResult> res(K);
  auto run = [&](size_t k) {
    int64_t from = k == 0 ? open + 1 : sp[k - 1];
    int64_t stop = k < sp.size() ? sp[k] : -1;
    res[k] = parse_slice(s, n, from, stop, k == 0, ap.chunks[k], elem);
  };
  pool_for(K, T, run);
  int64_t idx = 0;
  size_t used = 0;
  for (size_t k = 0; k < K; ++k) {
    ap.first_index.push_back(idx);
    idx += res[k].count;
    used = k + 1;
    if (res[k].syntax) { ap.syntax = true; ap.syntax_pos = res[k].syntax_pos; break; }
    if (res[k].end >= 0) { ap.end = res[k].end; break; }
    if (!res[k].reached_next) { ap.syntax = true; ap.syntax_pos = n; break; }
  }
  ap.chunks.resize(used);
  ap.first_index.resize(used);
  return ap;
}

}  // namespace

// ================================================================ handle

struct ks_trace {
  // events stay in the per-thread chunks they were parsed into; lmap / nmap
  // renumber chunk-local lane / name ids, ev_off[c] is chunk c's first row.
  int64_t n_events = 0;
  std::vector<EventChunk> ev;
  std::vector<int64_t> ev_off;
  std::vector<std::vector<int32_t>> lmap, nmap;
  std::vector<std::string> lanes;  // [0, n_event_lanes) == TraceColumns.from_events order
  int32_t n_event_lanes = 0;
  std::vector<std::string> names;
  // markers
  std::vector<int64_t> m_start, m_end;
  std::vector<int32_t> m_lane, m_layer;
  std::vector<uint8_t> m_phase;
  std::vector<std::string> layers;
  int64_t buckets_off = -1, buckets_len = 0, metadata_off = -1, metadata_len = 0;
  int32_t has_metadata = 0;
};

namespace {

template <class F>
void parallel_chunks(size_t n, F f) {
  if (n == 1) { f(0); return; }
  std::vector<std::thread> th;
  for (size_t c = 0; c < n; ++c) th.emplace_back(f, c);
  for (auto& x : th) x.join();
}

// global lane ids in TraceColumns.from_events order (event lanes by first
// appearance, then sync targets), names by first appearance.
void merge_events(ks_trace& t, std::vector<EventChunk>& chunks) {
  std::unordered_map<std::string, int32_t> gl;
  t.lmap.assign(chunks.size(), {});
  t.nmap.assign(chunks.size(), {});
  for (size_t c = 0; c < chunks.size(); ++c) t.lmap[c].assign(chunks[c].lanes.items.size(), -1);
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t c = 0; c < chunks.size(); ++c) {
      auto& ch = chunks[c];
      const auto& first = pass == 0 ? ch.lane_first_ev : ch.lane_first_sync;
      std::vector<int32_t> loc;
      for (size_t j = 0; j < first.size(); ++j)
        if (first[j] >= 0) loc.push_back((int32_t)j);
      std::sort(loc.begin(), loc.end(), [&](int32_t x, int32_t y) { return first[x] < first[y]; });
      for (int32_t j : loc) {
        if (t.lmap[c][(size_t)j] >= 0) continue;
        const std::string& s = ch.lanes.items[(size_t)j];
        auto it = gl.find(s);
        int32_t g;
        if (it == gl.end()) {
          g = (int32_t)t.lanes.size();
          gl.emplace(s, g);
          t.lanes.push_back(s);
        } else {
          g = it->second;
        }
        t.lmap[c][(size_t)j] = g;
      }
    }
  }
  t.n_event_lanes = (int32_t)t.lanes.size();
  std::unordered_map<std::string, int32_t> gn;
  for (size_t c = 0; c < chunks.size(); ++c) {
    auto& ch = chunks[c];
    t.nmap[c].resize(ch.names.items.size());
    for (size_t j = 0; j < ch.names.items.size(); ++j) {
      const std::string& s = ch.names.items[j];
      auto it = gn.find(s);
      if (it == gn.end()) {
        int32_t g = (int32_t)t.names.size();
        gn.emplace(s, g);
        t.names.push_back(s);
        t.nmap[c][j] = g;
      } else {
        t.nmap[c][j] = it->second;
      }
    }
  }
  t.ev_off.assign(chunks.size() + 1, 0);
  for (size_t c = 0; c < chunks.size(); ++c) t.ev_off[c + 1] = t.ev_off[c] + (int64_t)chunks[c].rows();
  t.n_events = t.ev_off.back();
  t.ev = std::move(chunks);
}

void merge_markers(ks_trace& t, std::vector<MarkerChunk>& chunks) {
  std::unordered_map<std::string, int32_t> gl, gy;
  for (int32_t j = 0; j < (int32_t)t.lanes.size(); ++j) gl.emplace(t.lanes[(size_t)j], j);
  for (auto& ch : chunks) {
    std::vector<int32_t> lm(ch.lanes.items.size()), ym(ch.layers.items.size());
    for (size_t j = 0; j < lm.size(); ++j) {
      auto it = gl.find(ch.lanes.items[j]);
      if (it == gl.end()) {
        lm[j] = (int32_t)t.lanes.size();
        gl.emplace(ch.lanes.items[j], lm[j]);
        t.lanes.push_back(ch.lanes.items[j]);
      } else {
        lm[j] = it->second;
      }
    }
    for (size_t j = 0; j < ym.size(); ++j) {
      auto it = gy.find(ch.layers.items[j]);
      if (it == gy.end()) {
        ym[j] = (int32_t)t.layers.size();
        gy.emplace(ch.layers.items[j], ym[j]);
        t.layers.push_back(ch.layers.items[j]);
      } else {
        ym[j] = it->second;
      }
    }
    for (size_t j = 0; j < ch.rows(); ++j) {
      t.m_start.push_back(ch.start[j]);
      t.m_end.push_back(ch.end[j]);
      t.m_lane.push_back(lm[(size_t)ch.lane[j]]);
      t.m_layer.push_back(ym[(size_t)ch.layer[j]]);
      t.m_phase.push_back(ch.phase[j]);
    }
  }
}

// first duplicate id in document order (trace.py:306-311)
bool first_duplicate(const ks_trace& t, int64_t& dup) {
  if (t.n_events < 2) return false;
  const size_t C = t.ev.size();
  {  // common case: ids strictly increasing in document order -> no duplicate
    std::vector<char> inc(C, 1);
    parallel_chunks(C, [&](size_t c) {
      const auto& v = t.ev[c].id;
      for (size_t j = 1; j < v.size(); ++j)
        if (v[j] <= v[j - 1]) { inc[c] = 0; return; }
    });
    bool ok = true;
    int64_t last = INT64_MIN;
    bool have = false;
    for (size_t c = 0; c < C && ok; ++c) {
      if (!inc[c]) { ok = false; break; }
      if (t.ev[c].id.empty()) continue;
      if (have && t.ev[c].id.front() <= last) ok = false;
      last = t.ev[c].id.back();
      have = true;
    }
    if (ok) return false;
  }
  std::vector<int64_t> los(C, INT64_MAX), his(C, INT64_MIN);
  parallel_chunks(C, [&](size_t c) {
    for (int64_t v : t.ev[c].id) { los[c] = std::min(los[c], v); his[c] = std::max(his[c], v); }
  });
  int64_t lo = *std::min_element(los.begin(), los.end());
  int64_t hi = *std::max_element(his.begin(), his.end());
  const int64_t n = t.n_events;
  if ((unsigned __int128)(hi - lo) < (unsigned __int128)n * 8 + 64) {
    int64_t range = hi - lo + 1;
    std::vector<std::atomic<uint64_t>> bits((size_t)((range + 63) / 64));
    for (auto& x : bits) x.store(0, std::memory_order_relaxed);
    std::atomic<bool> any{false};
    parallel_chunks(C, [&](size_t c) {
      for (int64_t v0 : t.ev[c].id) {
        uint64_t v = (uint64_t)(v0 - lo);
        uint64_t m = 1ull << (v & 63);
        if (bits[v >> 6].fetch_or(m, std::memory_order_relaxed) & m) { any = true; return; }
      }
    });
    if (!any) return false;
    std::vector<uint64_t> seen((size_t)((range + 63) / 64), 0);
    for (const auto& ch : t.ev)
      for (int64_t v0 : ch.id) {
        uint64_t v = (uint64_t)(v0 - lo);
        uint64_t m = 1ull << (v & 63);
        if (seen[v >> 6] & m) { dup = v0; return true; }
        seen[v >> 6] |= m;
      }
    return false;
  }
  std::vector<int64_t> srt;
  srt.reserve((size_t)n);
  for (const auto& ch : t.ev) srt.insert(srt.end(), ch.id.begin(), ch.id.end());
  std::sort(srt.begin(), srt.end());
  if (std::adjacent_find(srt.begin(), srt.end()) == srt.end()) return false;
  std::unordered_map<int64_t, char> seen;
  seen.reserve((size_t)n);
  for (const auto& ch : t.ev)
    for (int64_t v : ch.id)
      if (!seen.emplace(v, 1).second) { dup = v; return true; }
  return false;
}

// check_lane_overlaps (trace.py:255-265): per lane in first-appearance order,
// events ordered by (start, end, id); first adjacent pair with a.end > b.start.
bool first_overlap(const ks_trace& t, int T, int64_t& a_id, int64_t& b_id, int32_t& lane_out) {
  const int64_t n = t.n_events;
  const int32_t L = t.n_event_lanes;
  if (n < 2 || L == 0) return false;
  const size_t C = t.ev.size();
  // per (chunk, lane) counts -> offsets; scatter (start, end, id) per lane in document order
  std::vector<int64_t> cnt(C * (size_t)L, 0);
  parallel_chunks(C, [&](size_t c) {
    int64_t* k = &cnt[c * (size_t)L];
    for (int32_t l : t.ev[c].lane) ++k[t.lmap[c][(size_t)l]];
  });
  std::vector<int64_t> lane_ptr((size_t)L + 1, 0);
  std::vector<int64_t> off(C * (size_t)L);
  for (int32_t l = 0; l < L; ++l) {
    int64_t o = lane_ptr[(size_t)l];
    for (size_t c = 0; c < C; ++c) { off[c * (size_t)L + (size_t)l] = o; o += cnt[c * (size_t)L + (size_t)l]; }
    lane_ptr[(size_t)l + 1] = o;
  }
  struct Rec { int64_t start, end, id; };
  std::unique_ptr<Rec[]> rec(new Rec[(size_t)n]);
  parallel_chunks(C, [&](size_t c) {
    const auto& ch = t.ev[c];
    int64_t* o = &off[c * (size_t)L];
    for (size_t j = 0; j < ch.rows(); ++j) {
      int32_t l = t.lmap[c][(size_t)ch.lane[j]];
      rec[(size_t)o[l]++] = Rec{ch.start[j], ch.start[j] + ch.dur[j], ch.id[j]};
    }
  });
  auto less = [](const Rec& x, const Rec& y) {
    if (x.start != y.start) return x.start < y.start;
    if (x.end != y.end) return x.end < y.end;
    return x.id < y.id;
  };
  std::vector<int64_t> bad((size_t)L, -1);
  std::atomic<int32_t> next{0};
  auto worker = [&] {
    for (;;) {
      int32_t l = next++;
      if (l >= L) return;
      Rec* b = &rec[(size_t)lane_ptr[(size_t)l]];
      Rec* e = &rec[(size_t)lane_ptr[(size_t)l + 1]];
      if (!std::is_sorted(b, e, less)) std::sort(b, e, less);
      for (Rec* p = b; p + 1 < e; ++p)
        if (p[0].end > p[1].start) { bad[(size_t)l] = p - rec.get(); break; }
    }
  };
  int K = std::max(1, std::min(T, (int)L));
  std::vector<std::thread> th;
  for (int k = 0; k < K; ++k) th.emplace_back(worker);
  for (auto& x : th) x.join();
  for (int32_t l = 0; l < L; ++l) {
    if (bad[(size_t)l] >= 0) {
      a_id = rec[(size_t)bad[(size_t)l]].id;
      b_id = rec[(size_t)bad[(size_t)l] + 1].id;
      lane_out = l;
      return true;
    }
  }
  return false;
}

// check_marker_overlaps (trace.py:268-278): groups (layer, phase, lane) in
// first-appearance order, each sorted by start (stable).
bool marker_overlap(const ks_trace& t, std::string& msg) {
  size_t m = t.m_start.size();
  if (m < 2) return false;
  std::unordered_map<uint64_t, int32_t> gid;
  std::vector<int32_t> g(m);
  for (size_t i = 0; i < m; ++i) {
    uint64_t key = ((uint64_t)(uint32_t)t.m_layer[i] << 34) ^ ((uint64_t)t.m_phase[i] << 32) ^
                   (uint32_t)t.m_lane[i];
    auto it = gid.emplace(key, (int32_t)gid.size()).first;
    g[i] = it->second;
  }
  std::vector<int32_t> ord(m);
  for (size_t i = 0; i < m; ++i) ord[i] = (int32_t)i;
  std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
    if (g[a] != g[b]) return g[a] < g[b];
    return t.m_start[a] < t.m_start[b];
  });
  for (size_t j = 0; j + 1 < m; ++j) {
    int32_t a = ord[j], b = ord[j + 1];
    if (g[a] == g[b] && t.m_end[a] > t.m_start[b]) {
      msg = "overlapping markers for (" + t.layers[(size_t)t.m_layer[a]] + ", " +
            kPhaseNames[t.m_phase[a]] + ")";
      return true;
    }
  }
  return false;
}

int default_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h ? h : 1u, 64u));
}

}  // namespace

extern "C" {

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int ks_trace_parse(const char* text, int64_t len, int n_threads, ks_trace** out,
                   int64_t* err_ids) {
  const bool timing = std::getenv("DDSIM_TRACE_TIMING") != nullptr;
  double t0 = now_s();
  auto tick = [&](const char* what) {
    if (timing) { double t1 = now_s(); std::fprintf(stderr, "[ks_trace_parse] %-10s %.3f s\n", what, t1 - t0); t0 = t1; }
  };
  if (!text || len < 0 || !out) { set_last_error("ks_trace_parse: bad arguments"); return KS_ERR_INVALID; }
  *out = nullptr;
  int T = n_threads > 0 ? std::min(n_threads, 256) : default_threads();
  if (n_threads <= 0 && len < (4 << 20)) T = 1;  // explicit counts are honoured (tests)
  auto t = new ks_trace();
  Err syntax, top, ev, evdoc, mk, mkdoc;
  PreScan ps;
  bool scanned = false;
  auto need_scan = [&] {
    if (!scanned && T > 1) {
      // ~2 MB chunks (at least 4 per thread, at most 4096)
      const int64_t k0 = std::max<int64_t>((int64_t)T * 4, std::min<int64_t>(4096, len >> 21));
      ps = prescan(text, len, (int)k0, T);
      scanned = true;
    }
  };

  Lexer L(text, text + len, text);
  L.ws();
  Val ver, unit, events_v, markers_v;
  std::vector<EventChunk> ev_chunks;
  std::vector<int64_t> ev_first;
  std::vector<MarkerChunk> mk_chunks;
  std::vector<int64_t> mk_first;

  auto array_of = [&](auto elem, auto& chunks, auto& first, int64_t open) -> bool {
    using ChunkT = typename std::decay_t<decltype(chunks)>::value_type;
    std::vector<int64_t> sp;
    if (T > 1) {
      need_scan();
      sp = split_points(ps, open);
      tick("split");
    }
    auto ap = parse_array<ChunkT>(text, len, open, sp, elem, T);
    if (ap.syntax) {
      L.cur = text + std::max<int64_t>(ap.syntax_pos, 0);
      L.fail();
      return false;
    }
    chunks = std::move(ap.chunks);
    first = std::move(ap.first_index);
    tick("array");
    L.cur = text + ap.end;
    return true;
  };

  if (L.peek() != '{') {
    Val v;
    if (L.value(v)) {
      L.ws();
      if (L.cur != L.e) L.fail();
    }
    if (L.bad) syntax.set(E_MALFORMED, "invalid JSON at offset " + std::to_string(L.badpos - text));
    else top.set(E_MALFORMED, "top-level value must be an object");
  } else {
    ++L.cur;
    L.ws();
    if (L.peek() == '}') {
      ++L.cur;
    } else {
      for (;;) {
        L.ws();
        Val k;
        if (L.peek() != '"' || !L.string(k)) { L.fail(); break; }
        L.ws();
        if (L.peek() != ':') { L.fail(); break; }
        ++L.cur;
        L.ws();
        std::string key = unescape(k);
        const char* vstart = L.cur;
        if (key == "events" && L.peek() == '[') {
          // last occurrence wins (json.loads keeps the last duplicate key)
          ev_chunks.clear();
          if (!array_of(event_element, ev_chunks, ev_first, L.cur - text)) break;
          events_v.t = V_ARR;
        } else if (key == "layer_markers" && L.peek() == '[') {
          mk_chunks.clear();
          if (!array_of(marker_element, mk_chunks, mk_first, L.cur - text)) break;
          markers_v.t = V_ARR;
        } else {
          Val v;
          if (!L.value(v)) break;
          if (key == "schema_version") ver = v;
          else if (key == "time_unit") unit = v;
          else if (key == "events") { events_v = v; ev_chunks.clear(); }
          else if (key == "layer_markers") { markers_v = v; mk_chunks.clear(); }
          else if (key == "gradient_buckets") {
            t->buckets_off = vstart - text;
            t->buckets_len = L.cur - vstart;
          } else if (key == "metadata") {
            t->metadata_off = vstart - text;
            t->metadata_len = L.cur - vstart;
            t->has_metadata = 1;
          }
        }
        L.ws();
        int c = L.peek();
        if (c == ',') { ++L.cur; continue; }
        if (c == '}') { ++L.cur; break; }
        L.fail();
        break;
      }
    }
    if (!L.bad) {
      L.ws();
      if (L.cur != L.e) L.fail();  // "Extra data"
    }
    if (L.bad) syntax.set(E_MALFORMED, "invalid JSON at offset " + std::to_string(L.badpos - text));
  }

  tick("parse");
  int rc = KS_OK;
  auto finish = [&](int code, const std::string& msg) {
    set_last_error(msg);
    rc = code;
  };
  if (syntax.code) {
    finish(syntax.code, syntax.msg);
  } else if (top.code) {
    finish(top.code, top.msg);
  } else if (ver.t == V_ABSENT) {
    finish(E_SCHEMA, "document: missing field 'schema_version'");
  } else if (!((ver.t == V_INT || ver.t == V_FLOAT) &&
               [&] { Dec d; if (ver.t == V_FLOAT && !float_repr_dec(ver, d)) return false;
                     if (ver.t == V_INT) literal_dec(ver.p, ver.n, d);
                     return !d.neg && d.digits == "1" && d.exp == 0; }()) &&
             ver.t != V_TRUE) {
    finish(E_SCHEMA, "unsupported schema_version " + val_repr(ver));
  } else if (unit.t == V_ABSENT) {
    finish(E_SCHEMA, "document: missing field 'time_unit'");
  } else if (!str_eq(unit, "microseconds")) {
    finish(E_SCHEMA, "unsupported time_unit " + val_repr(unit));
  } else if (events_v.t != V_ABSENT && events_v.t != V_ARR) {
    finish(E_SCHEMA, "events must be an array");
  }
  if (rc == KS_OK) {
    for (size_t c = 0; c < ev_chunks.size(); ++c) {
      if (ev_chunks[c].err.code) {
        int64_t idx = ev_first[c] + ev_chunks[c].err_row;
        finish(ev_chunks[c].err.code,
               with_ctx("events[" + std::to_string(idx) + "]", ev_chunks[c].err.msg));
        break;
      }
    }
  }
  int T2 = n_threads > 0 ? std::min(n_threads, 256) : default_threads();
  if (rc == KS_OK) {
    merge_events(*t, ev_chunks);
    tick("merge");
    int64_t dup;
    int64_t a, b;
    int32_t ln;
    bool has_dup = first_duplicate(*t, dup);
    tick("dup-ids");
    if (has_dup) {
      finish(E_SCHEMA, "duplicate event id " + std::to_string(dup));
    } else if (first_overlap(*t, T2, a, b, ln)) {
      finish(E_OVERLAP, "events " + std::to_string(a) + " and " + std::to_string(b) +
                            " overlap on lane " + t->lanes[(size_t)ln]);
      if (err_ids) { err_ids[0] = a; err_ids[1] = b; }
    }
  }
  if (rc == KS_OK && markers_v.t != V_ABSENT && markers_v.t != V_ARR)
    finish(E_SCHEMA, "layer_markers must be an array");
  if (rc == KS_OK) {
    for (size_t c = 0; c < mk_chunks.size(); ++c) {
      if (mk_chunks[c].err.code) {
        int64_t idx = mk_first[c] + mk_chunks[c].err_row;
        finish(mk_chunks[c].err.code,
               with_ctx("layer_markers[" + std::to_string(idx) + "]", mk_chunks[c].err.msg));
        break;
      }
    }
  }
  if (rc == KS_OK) {
    tick("overlaps");
    merge_markers(*t, mk_chunks);
    std::string msg;
    if (marker_overlap(*t, msg)) finish(E_SCHEMA, msg);
    tick("markers");
  }
  if (rc != KS_OK) {
    delete t;
    return rc;
  }
  *out = t;
  return KS_OK;
}

int ks_trace_get_info(const ks_trace* t, ks_trace_info* info) {
  if (!t || !info) return KS_ERR_INVALID;
  info->n_events = t->n_events;
  info->n_lanes = (int32_t)t->lanes.size();
  info->n_event_lanes = t->n_event_lanes;
  info->n_names = (int64_t)t->names.size();
  info->n_markers = (int64_t)t->m_start.size();
  info->n_layers = (int32_t)t->layers.size();
  auto bytes = [](const std::vector<std::string>& v) {
    int64_t s = 0;
    for (auto& x : v) s += (int64_t)x.size();
    return s;
  };
  info->lane_bytes = bytes(t->lanes);
  info->name_bytes = bytes(t->names);
  info->layer_bytes = bytes(t->layers);
  info->buckets_off = t->buckets_off;
  info->buckets_len = t->buckets_len;
  info->metadata_off = t->metadata_off;
  info->metadata_len = t->metadata_len;
  return KS_OK;
}

int ks_trace_events(const ks_trace* t, const ks_trace_event_cols* c) {
  if (!t || !c) return KS_ERR_INVALID;
  parallel_chunks(t->ev.size(), [&](size_t k) {
    const auto& ch = t->ev[k];
    size_t m = ch.rows();
    int64_t o = t->ev_off[k];
    if (!m) return;
    auto cp = [&](void* dst, const void* src, size_t w) {
      if (dst) std::memcpy((char*)dst + (size_t)o * w, src, m * w);
    };
    cp(c->id, ch.id.data(), 8);
    cp(c->kind, ch.kind.data(), 1);
    cp(c->start, ch.start.data(), 8);
    cp(c->duration, ch.dur.data(), 8);
    cp(c->correlation, ch.corr.data(), 8);
    cp(c->is_dtoh, ch.dtoh.data(), 1);
    cp(c->size_bytes, ch.size.data(), 8);
    const auto& lm = t->lmap[k];
    const auto& nm = t->nmap[k];
    if (c->lane)
      for (size_t j = 0; j < m; ++j) c->lane[(size_t)o + j] = lm[(size_t)ch.lane[j]];
    if (c->sync_target)
      for (size_t j = 0; j < m; ++j)
        c->sync_target[(size_t)o + j] = ch.sync[j] < 0 ? -1 : lm[(size_t)ch.sync[j]];
    if (c->name_id)
      for (size_t j = 0; j < m; ++j) c->name_id[(size_t)o + j] = nm[(size_t)ch.name[j]];
  });
  return KS_OK;
}

int ks_trace_markers(const ks_trace* t, const ks_trace_marker_cols* c) {
  if (!t || !c) return KS_ERR_INVALID;
  size_t m = t->m_start.size();
  auto cp = [m](void* dst, const void* src, size_t w) {
    if (dst && m) std::memcpy(dst, src, m * w);
  };
  cp(c->lane, t->m_lane.data(), 4);
  cp(c->start, t->m_start.data(), 8);
  cp(c->end, t->m_end.data(), 8);
  cp(c->layer_id, t->m_layer.data(), 4);
  cp(c->phase, t->m_phase.data(), 1);
  return KS_OK;
}

int ks_trace_strings(const ks_trace* t, int which, char* bytes, int64_t* offsets) {
  if (!t) return KS_ERR_INVALID;
  const std::vector<std::string>* v = which == 0 ? &t->lanes : which == 1 ? &t->names
                                    : which == 2 ? &t->layers : nullptr;
  if (!v) return KS_ERR_INVALID;
  int64_t o = 0;
  for (size_t i = 0; i < v->size(); ++i) {
    if (offsets) offsets[i] = o;
    if (bytes) std::memcpy(bytes + o, (*v)[i].data(), (*v)[i].size());
    o += (int64_t)(*v)[i].size();
  }
  if (offsets) offsets[v->size()] = o;
  return KS_OK;
}

void ks_trace_destroy(ks_trace* t) { delete t; }

}  // extern "C"

// ================================================================ writer
//
// Columns -> trace document text (the inverse of ks_trace_parse, for traces
// too large for kernsim.trace.dump_trace, trace.py:331-379).  Times use
// ns_to_us_number (trace.py:101-105): integer microseconds when exact, else
// Python's repr of float(Decimal(ns) / 1000); strings are escaped like
// json.dumps (ensure_ascii).

namespace {

void put_json_string(std::string& o, const char* p, int64_t n) {
  static const char* hex = "0123456789abcdef";
  auto u16 = [&](uint32_t v) {
    o += "\\u";
    o += hex[(v >> 12) & 15]; o += hex[(v >> 8) & 15]; o += hex[(v >> 4) & 15]; o += hex[v & 15];
  };
  o += '"';
  const unsigned char* s = (const unsigned char*)p;
  const unsigned char* e = s + n;
  while (s < e) {
    unsigned char c = *s;
    if (c < 0x80) {
      switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        default:
          if (c < 0x20) u16(c); else o += (char)c;
      }
      ++s;
      continue;
    }
    uint32_t cp;
    int len;
    if ((c & 0xE0) == 0xC0) { cp = c & 0x1F; len = 2; }
    else if ((c & 0xF0) == 0xE0) { cp = c & 0x0F; len = 3; }
    else { cp = c & 0x07; len = 4; }
    for (int k = 1; k < len && s + k < e; ++k) cp = (cp << 6) | (s[k] & 0x3F);
    s += len;
    if (cp >= 0x10000) {
      cp -= 0x10000;
      u16(0xD800 + (cp >> 10));
      u16(0xDC00 + (cp & 0x3FF));
    } else {
      u16(cp);
    }
  }
  o += '"';
}

void put_us(std::string& o, int64_t ns) {
  char buf[64];
  if (ns % 1000 == 0) {
    auto r = std::to_chars(buf, buf + sizeof buf, ns / 1000);
    o.append(buf, r.ptr);
    return;
  }
  // exact decimal ns/1000 -> nearest double -> shortest repr (fixed)
  bool neg = ns < 0;
  unsigned long long m = neg ? 0ull - (unsigned long long)ns : (unsigned long long)ns;
  std::string d = std::to_string(m);
  while (d.size() < 4) d.insert(d.begin(), '0');
  std::string lit = (neg ? "-" : "") + d.substr(0, d.size() - 3) + "." + d.substr(d.size() - 3);
  double x = std::strtod(lit.c_str(), nullptr);
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::fixed);
  std::string_view sv(buf, (size_t)(r.ptr - buf));
  o.append(sv);
  if (sv.find('.') == std::string_view::npos) o += ".0";
}

inline void put_i64(std::string& o, int64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  o.append(buf, r.ptr);
}

}  // namespace

extern "C" {

int ks_trace_write(const ks_trace_write_desc* d, int n_threads, char** out, int64_t* out_len) {
  if (!d || !out || !out_len) { set_last_error("ks_trace_write: bad arguments"); return KS_ERR_INVALID; }
  *out = nullptr;
  *out_len = 0;
  int T = n_threads > 0 ? std::min(n_threads, 256) : default_threads();
  auto str_of = [](const char* bytes, const int64_t* off, int64_t i) {
    return std::string_view(bytes + off[i], (size_t)(off[i + 1] - off[i]));
  };
  for (int64_t i = 0; i < d->n_events; ++i) {
    if (d->kind[i] >= kKinds || d->lane[i] < 0 || d->lane[i] >= d->n_lanes ||
        d->name_id[i] < 0 || d->name_id[i] >= d->n_names ||
        (d->sync_target && d->sync_target[i] >= d->n_lanes)) {
      set_last_error("ks_trace_write: event " + std::to_string(i) + " has an out-of-range code");
      return KS_ERR_INVALID;
    }
  }
  // pre-escaped lane / name / layer strings
  auto escaped = [&](const char* bytes, const int64_t* off, int64_t n) {
    std::vector<std::string> v((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      auto s = str_of(bytes, off, i);
      put_json_string(v[(size_t)i], s.data(), (int64_t)s.size());
    }
    return v;
  };
  auto lanes = escaped(d->lane_bytes, d->lane_off, d->n_lanes);
  auto names = escaped(d->name_bytes, d->name_off, d->n_names);
  auto layers = escaped(d->layer_bytes, d->layer_off, d->n_layers);

  auto events_part = [&](int64_t b, int64_t e, std::string& o) {
    o.reserve((size_t)(e - b) * 150);
    for (int64_t i = b; i < e; ++i) {
      if (i) o += ", ";
      o += "{\"id\": ";
      put_i64(o, d->id[i]);
      o += ", \"kind\": \"";
      o += kKindNames[d->kind[i]];
      o += "\", \"name\": ";
      o += names[(size_t)d->name_id[i]];
      o += ", \"lane\": ";
      o += lanes[(size_t)d->lane[i]];
      o += ", \"start\": ";
      put_us(o, d->start[i]);
      o += ", \"duration\": ";
      put_us(o, d->duration[i]);
      if (d->correlation && d->correlation[i] >= 0) {
        o += ", \"correlation\": ";
        put_i64(o, d->correlation[i]);
      }
      if (d->size_bytes && d->size_bytes[i] >= 0) {
        o += ", \"size_bytes\": ";
        put_i64(o, d->size_bytes[i]);
      }
      if (d->sync_target && d->sync_target[i] >= 0) {
        o += ", \"sync_target\": ";
        o += lanes[(size_t)d->sync_target[i]];
      }
      o += "}";
    }
  };
  auto markers_part = [&](int64_t b, int64_t e, std::string& o) {
    o.reserve((size_t)(e - b) * 110);
    for (int64_t i = b; i < e; ++i) {
      if (i) o += ", ";
      o += "{\"layer\": ";
      o += layers[(size_t)d->m_layer[i]];
      o += ", \"phase\": \"";
      o += kPhaseNames[d->m_phase[i] % 3];
      o += "\", \"cpu_lane\": ";
      o += lanes[(size_t)d->m_lane[i]];
      o += ", \"start\": ";
      put_us(o, d->m_start[i]);
      o += ", \"end\": ";
      put_us(o, d->m_end[i]);
      o += "}";
    }
  };
  auto chunked = [&](int64_t n, auto part) {
    int K = (int)std::max<int64_t>(1, std::min<int64_t>(T, n / 16384 + 1));
    std::vector<std::string> parts((size_t)K);
    int64_t step = (n + K - 1) / K;
    std::vector<std::thread> th;
    for (int k = 0; k < K; ++k) {
      int64_t b = std::min(n, (int64_t)k * step), e = std::min(n, b + step);
      th.emplace_back([&, k, b, e] { part(b, e, parts[(size_t)k]); });
    }
    for (auto& x : th) x.join();
    return parts;
  };
  auto ev = chunked(d->n_events, events_part);
  auto mk = chunked(d->n_markers, markers_part);
  std::string head = "{\"schema_version\": 1, \"time_unit\": \"microseconds\", \"events\": [";
  std::string mid = "], \"layer_markers\": [";
  std::string tail = "]";
  if (d->extra_json && *d->extra_json) { tail += ", "; tail += d->extra_json; }
  tail += "}";
  size_t total = head.size() + mid.size() + tail.size();
  for (auto& p : ev) total += p.size();
  for (auto& p : mk) total += p.size();
  char* buf = (char*)std::malloc(total + 1);
  if (!buf) { set_last_error("ks_trace_write: out of host memory"); return KS_ERR_OOM; }
  size_t o = 0;
  auto put = [&](const std::string& s) { std::memcpy(buf + o, s.data(), s.size()); o += s.size(); };
  put(head);
  for (auto& p : ev) put(p);
  put(mid);
  for (auto& p : mk) put(p);
  put(tail);
  buf[o] = 0;
  *out = buf;
  *out_len = (int64_t)o;
  return KS_OK;
}

void ks_buffer_free(char* p) { std::free(p); }

}  // extern "C"
