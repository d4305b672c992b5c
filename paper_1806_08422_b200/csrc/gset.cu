// Native G-set / edge-list instance parser (parse_gset, gset.py:35-89).
//
// Host code (no kernels): the reference parses a K2000-size file (2M edge
// lines) in ~6.5 s of Python; this single pass over the bytes
// plus a sort for duplicate detection takes tens of milliseconds.  Semantics
// follow gset.py exactly:
//  * lines split like str.splitlines() for ASCII text (\n, \r\n, \r, \v, \f,
//    \x1c-\x1e), stripped; empty lines and lines starting with '#' or 'c' are
//    comments;
//  * header "n m" (2 tokens, integers, n >= 1, m >= 0);
//  * edge lines "u v w" (3 tokens, u, v integers in [1, n], u != v, w finite
//    and nonzero, no duplicate unordered pair, at most m lines, exactly m);
//  * the FIRST failing line in file order is reported, with the reference's
//    message text and 1-based line number.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.h"

namespace nmfa {
namespace {

bool is_line_break(unsigned char c) {
  return c == '\n' || c == '\r' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e;
}
bool is_space(unsigned char c) {  // str.split() / str.strip() whitespace (ASCII)
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' ||
         (c >= 0x1c && c <= 0x1f);
}

struct Token {
  const char* p;
  size_t n;
  std::string str() const { return std::string(p, n); }
};

// Python repr of a list of str tokens (printable ASCII without quotes/backslashes
// is the common case; other characters are escaped the way repr() does).
std::string py_list_repr(const std::vector<Token>& t) {
  std::string s = "[";
  for (size_t k = 0; k < t.size(); ++k) {
    if (k) s += ", ";
    const std::string v = t[k].str();
    const bool has_sq = v.find('\'') != std::string::npos, has_dq = v.find('"') != std::string::npos;
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    s += q;
    for (unsigned char c : v) {
      if (c == '\\') s += "\\\\";
      else if (c == (unsigned char)q) { s += '\\'; s += (char)c; }
      else if (c == '\t') s += "\\t";
      else if (c < 0x20 || c == 0x7f) {
        char buf[8];
        snprintf(buf, sizeof buf, "\\x%02x", c);
        s += buf;
      } else s += (char)c;  // printable ASCII and UTF-8 bytes pass through
    }
    s += q;
  }
  return s + "]";
}

// Python int(): optional sign, ASCII digits with single underscores between digits.
bool parse_int(const Token& t, long long* out) {
  size_t i = 0;
  bool neg = false;
  if (i < t.n && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
  if (i >= t.n) return false;
  long long v = 0;
  bool prev_digit = false, big = false;
  for (; i < t.n; ++i) {
    const char c = t.p[i];
    if (c >= '0' && c <= '9') {
      if (v > (LLONG_MAX - 9) / 10) big = true;  // a valid Python int beyond int64
      else v = v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < t.n && t.p[i + 1] >= '0' && t.p[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  if (big) v = LLONG_MAX;  // fails every range check, like the reference's huge ints
  *out = neg ? -v : v;
  return true;
}

// Python float(): decimal / exponent forms, inf / infinity / nan (any case),
// underscores between digits.
bool parse_float(const Token& t, double* out) {
  {  // fast path: a plain decimal integer (the common G-set weight), exact
    size_t i = 0;
    bool neg = false;
    if (i < t.n && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    if (i < t.n && t.n - i <= 15) {
      long long v = 0;
      size_t j = i;
      for (; j < t.n && t.p[j] >= '0' && t.p[j] <= '9'; ++j) v = v * 10 + (t.p[j] - '0');
      if (j == t.n) {
        *out = neg ? -(double)v : (double)v;
        return true;
      }
    }
  }
  std::string s;
  s.reserve(t.n);
  for (size_t i = 0; i < t.n; ++i) {
    const char c = t.p[i];
    if (c == '_') {
      const bool ok = i > 0 && i + 1 < t.n && std::isdigit((unsigned char)t.p[i - 1]) &&
                      std::isdigit((unsigned char)t.p[i + 1]);
      if (!ok) return false;
      continue;
    }
    s += c;
  }
  if (s.empty()) return false;
  std::string low;
  for (char c : s) low += (char)std::tolower((unsigned char)c);
  size_t k = (low[0] == '+' || low[0] == '-') ? 1 : 0;
  const std::string body = low.substr(k);
  if (body == "inf" || body == "infinity" || body == "nan") {
    *out = body == "nan" ? NAN : (low[0] == '-' ? -INFINITY : INFINITY);
    return true;
  }
  // strtod accepts hex floats and leading whitespace; Python float() does not
  if (body.find('x') != std::string::npos || body.empty()) return false;
  for (char c : body)
    if (!(std::isdigit((unsigned char)c) || c == '.' || c == 'e' || c == '+' || c == '-')) return false;
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) return false;
  *out = v;  // overflow gives +-inf like Python (float('1e999') == inf)
  return true;
}

struct Parser {
  const char* text;
  size_t len, pos = 0;
  long long line_no = 0;
  bool next_line(std::vector<Token>& toks) {  // next content line; false at EOF
    while (pos < len) {
      const size_t start = pos;
      while (pos < len && !is_line_break((unsigned char)text[pos])) ++pos;
      size_t end = pos;
      if (pos < len) {  // consume the break (\r\n counts once)
        if (text[pos] == '\r' && pos + 1 < len && text[pos + 1] == '\n') ++pos;
        ++pos;
      }
      ++line_no;
      size_t a = start, b = end;
      while (a < b && is_space((unsigned char)text[a])) ++a;
      while (b > a && is_space((unsigned char)text[b - 1])) --b;
      if (a == b || text[a] == '#' || text[a] == 'c') continue;
      toks.clear();
      size_t i = a;
      while (i < b) {
        while (i < b && is_space((unsigned char)text[i])) ++i;
        const size_t s = i;
        while (i < b && !is_space((unsigned char)text[i])) ++i;
        if (i > s) toks.push_back({text + s, i - s});
      }
      return true;
    }
    return false;
  }
};

int fail(long long line_no, const std::string& msg) {
  set_error("line " + std::to_string(line_no) + ": " + msg);
  return NMFA_ERR_ARG;
}

}  // namespace

int gset_parse(const char* text, int64_t len, int64_t* n_out, int64_t* m_out, int64_t* ei,
               int64_t* ej, double* w, int64_t cap) {
  Parser ps{text, (size_t)len};
  std::vector<Token> t;
  if (!ps.next_line(t)) return fail(0, "empty instance: missing header");
  if (t.size() != 2)
    return fail(ps.line_no, "header must be 'n m', got " + std::to_string(t.size()) + " tokens");
  long long n = 0, m = 0;
  if (!parse_int(t[0], &n) || !parse_int(t[1], &m))
    return fail(ps.line_no, "non-numeric header token in " + py_list_repr(t));
  if (n < 1) return fail(ps.line_no, "vertex count must be positive, got " + std::to_string(n));
  if (m < 0) return fail(ps.line_no, "edge count must be nonnegative, got " + std::to_string(m));
  if (n > (1LL << 30)) return fail(ps.line_no, "vertex count too large, got " + std::to_string(n));
  *n_out = n;
  *m_out = m;
  if (!ei) return NMFA_OK;  // header query
  if (cap < m) {
    set_error("output arrays hold fewer than the declared edge count");
    return NMFA_ERR_ARG;
  }
  // one pass in file order; duplicates are resolved afterwards by a sort, and
  // the earliest failure (parse error or duplicate) wins
  // duplicates: an n x n bitset checked in file order when it is small
  // (<= 64 MB, n <~ 23k), else one sort after the pass
  // (n <= 23170 keeps n * n far from 64-bit overflow; larger n sorts)
  const bool use_bits = n <= 23170 && (unsigned long long)n * (unsigned long long)n <= (64ULL << 23);
  std::vector<uint64_t> seen(use_bits ? ((unsigned long long)n * n + 63) / 64 : 0, 0);
  std::vector<long long> line_of;
  line_of.reserve((size_t)std::min<long long>(m, (long long)len / 4 + 1));  // m may be absurd
  long long count = 0, last_line = ps.line_no, err_line = -1;
  std::string err_msg;
  while (ps.next_line(t)) {
    last_line = ps.line_no;
    std::string msg;
    long long u = 0, v = 0;
    double wt = 0.0;
    if (t.size() != 3) {
      msg = "edge line must be 'u v w', got " + std::to_string(t.size()) + " tokens";
    } else if (!parse_int(t[0], &u) || !parse_int(t[1], &v) || !parse_float(t[2], &wt)) {
      msg = "non-numeric token in " + py_list_repr(t);
    } else if (!(1 <= u && u <= n) || !(1 <= v && v <= n)) {
      msg = "vertex index out of range [1, " + std::to_string(n) + "]";
    } else if (u == v) {
      msg = "self-loop at vertex " + std::to_string(u);
    } else if (wt == 0.0 || !std::isfinite(wt)) {
      msg = "edge weight must be finite and nonzero, got " + t[2].str();
    } else if (use_bits && ((seen[((uint64_t)(std::min(u, v) - 1) * n + (std::max(u, v) - 1)) >> 6] >>
                             (((uint64_t)(std::min(u, v) - 1) * n + (std::max(u, v) - 1)) & 63)) & 1)) {
      msg = "duplicate edge (" + std::to_string(std::min(u, v)) + ", " + std::to_string(std::max(u, v)) + ")";
    } else if (count >= m) {
      // the reference tests for a duplicate before the count (gset.py:75-80)
      const long long a = std::min(u, v) - 1, b = std::max(u, v) - 1;
      for (long long k = 0; k < count && msg.empty(); ++k)
        if (std::min(ei[k], ej[k]) == a && std::max(ei[k], ej[k]) == b)
          msg = "duplicate edge (" + std::to_string(a + 1) + ", " + std::to_string(b + 1) + ")";
      if (msg.empty()) msg = "more edge lines than the declared " + std::to_string(m);
    }
    if (!msg.empty()) {
      err_line = ps.line_no;
      err_msg = msg;
      break;
    }
    ei[count] = u - 1;
    ej[count] = v - 1;
    w[count] = wt;
    if (use_bits) {
      const uint64_t bit = (uint64_t)(std::min(u, v) - 1) * n + (std::max(u, v) - 1);
      seen[bit >> 6] |= 1ULL << (bit & 63);
    } else {
      line_of.push_back(ps.line_no);
    }
    ++count;
  }
  // first duplicate unordered pair in file order (the second occurrence's line)
  long long dup_line = -1;
  std::string dup_msg;
  if (!use_bits && count > 1) {
    std::vector<int64_t> order((size_t)count);
    for (int64_t k = 0; k < count; ++k) order[k] = k;
    auto key = [&](int64_t k) {
      const int64_t a = std::min(ei[k], ej[k]), b = std::max(ei[k], ej[k]);
      return (uint64_t)a * (uint64_t)n + (uint64_t)b;
    };
    std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
      const uint64_t kx = key(x), ky = key(y);
      return kx != ky ? kx < ky : x < y;
    });
    for (int64_t k = 1; k < count; ++k) {
      if (key(order[k]) == key(order[k - 1])) {
        const int64_t later = order[k];  // a repeat of an earlier line
        if (dup_line < 0 || line_of[later] < dup_line) {
          dup_line = line_of[later];
          const int64_t a = std::min(ei[later], ej[later]) + 1, b = std::max(ei[later], ej[later]) + 1;
          dup_msg = "duplicate edge (" + std::to_string(a) + ", " + std::to_string(b) + ")";
        }
      }
    }
  }
  if (dup_line >= 0 && (err_line < 0 || dup_line < err_line)) return fail(dup_line, dup_msg);
  if (err_line >= 0) return fail(err_line, err_msg);
  if (count != m)
    return fail(last_line, "header declared " + std::to_string(m) + " edges but found " +
                               std::to_string(count));
  return NMFA_OK;
}

}  // namespace nmfa
