// rqa_ingest.cpp -- native, multi-threaded read_column (tiledrqa ingest.py:53-129).
//
// Semantics of the reference, for ASCII files:
//   * lines end at "\r\n", "\r" or "\n" (Python text mode, universal newlines);
//     line numbers are 1-based physical lines;
//   * empty lines are ignored and do not count toward `offset`; the first
//     `offset` non-empty lines are skipped unparsed;
//   * the row is split on the delimiter; a row without the requested column
//     is ColumnOutOfRange (or skipped with skip_invalid);
//   * the token is str.strip()ped and parsed like float(): optional sign,
//     digits with single underscores between digits, optional fraction,
//     optional exponent, or inf / infinity / nan (any case); anything else,
//     and any non-finite value, is ParseError (or skipped).
// Files containing a byte >= 0x80 (non-ASCII UTF-8: Unicode whitespace and
// digits change float()'s behaviour) return RQA_EUNSUPPORTED so that the
// caller uses its Python implementation.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rqa_b200.h"

namespace {

void ing_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

// str.strip() / float() whitespace in the ASCII range
inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

inline bool ieq(const char* a, size_t n, const char* lit) {
  if (strlen(lit) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if ((a[i] | 0x20) != lit[i]) return false;
  return true;
}

// Digits with single underscores between digits.  Returns the number of
// characters consumed (0 if no digit at p); *under is set when an
// underscore was seen.
inline size_t py_digits(const char* p, const char* e, bool* under) {
  const char* q = p;
  if (q >= e || !(*q >= '0' && *q <= '9')) return 0;
  while (q < e) {
    if (*q >= '0' && *q <= '9') {
      ++q;
    } else if (*q == '_' && q + 1 < e && q[1] >= '0' && q[1] <= '9' && q > p) {
      *under = true;
      ++q;
    } else {
      break;
    }
  }
  return (size_t)(q - p);
}

// Characters strtod could read past the end of a validated token.
inline bool strtod_may_continue(char c) {
  return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') ||
         c == '.' || c == '+' || c == '-' || c == '_';
}

// float(token) for an already stripped ASCII token; false on ValueError.
// `limit` is the end of readable memory (for parsing in place).
bool py_float(const char* p, size_t n, const char* limit, double* out, std::string& buf) {
  if (n == 0) return false;
  const char* e = p + n;
  const char* q = p;
  bool neg = false;
  if (*q == '+' || *q == '-') {
    neg = *q == '-';
    ++q;
  }
  const size_t rest = (size_t)(e - q);
  if (rest >= 3 && rest <= 8 && (ieq(q, rest, "inf") || ieq(q, rest, "infinity"))) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(q, rest, "nan")) {
    *out = NAN;
    return true;
  }
  // grammar of float(): digits [. digits] [e [sign] digits], underscores between digits
  bool under = false;
  const size_t ni = py_digits(q, e, &under);
  q += ni;
  size_t nf = 0;
  if (q < e && *q == '.') {
    ++q;
    nf = py_digits(q, e, &under);
    q += nf;
  }
  if (ni == 0 && nf == 0) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    const size_t ne = py_digits(q, e, &under);
    if (ne == 0) return false;
    q += ne;
  }
  if (q != e) return false;
  // correctly rounded conversion (glibc strtod); overflow gives +-inf
  if (!under && e < limit && !strtod_may_continue(*e)) {
    char* end = nullptr;
    const double v = strtod(p, &end);
    if (end == e) {
      *out = v;
      return true;
    }
  }
  buf.clear();
  for (const char* c = p; c < e; ++c)
    if (*c != '_') buf.push_back(*c);
  *out = strtod(buf.c_str(), nullptr);
  return true;
}

struct Line {
  const char* p;
  size_t n;
};

// Line boundaries of [b, e): "\r\n", "\r" and "\n" each end a line.
inline const char* next_line(const char* p, const char* e, Line* ln) {
  const char* q = p;
  while (q < e && *q != '\n' && *q != '\r') ++q;
  ln->p = p;
  ln->n = (size_t)(q - p);
  if (q < e) {
    if (*q == '\r' && q + 1 < e && q[1] == '\n') q += 2;
    else ++q;
  }
  return q;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0, nonempty = 0;  // pass 1
  int64_t line0 = 0, skip = 0;      // first physical line number - 1, offset rows inside
  std::vector<double> vals;         // pass 2
  int64_t skipped = 0;
  int64_t err_line = 0;             // first error (0: none)
  int err_kind = 0;                 // 1 column out of range, 2 parse error
  int64_t err_fields = 0;
  std::string err_token;
};

void count_lines(Chunk* c) {
  Line ln;
  for (const char* p = c->b; p < c->e;) {
    p = next_line(p, c->e, &ln);
    ++c->lines;
    c->nonempty += ln.n > 0;
  }
}

void parse_chunk(Chunk* c, const char* limit, char delim, int64_t column, int skip_invalid) {
  Line ln;
  std::string buf;
  int64_t lineno = c->line0, skip = c->skip;
  for (const char* p = c->b; p < c->e;) {
    p = next_line(p, c->e, &ln);
    ++lineno;
    if (ln.n == 0) continue;
    if (skip > 0) {
      --skip;
      continue;
    }
    // field `column` of the row
    const char* f = ln.p;
    const char* le = ln.p + ln.n;
    int64_t idx = 0;
    while (idx < column) {
      const char* d = (const char*)memchr(f, delim, (size_t)(le - f));
      if (!d) break;
      f = d + 1;
      ++idx;
    }
    if (idx < column) {
      if (skip_invalid) {
        ++c->skipped;
        continue;
      }
      c->err_line = lineno;
      c->err_kind = 1;
      c->err_fields = idx + 1;
      return;
    }
    const char* fe = (const char*)memchr(f, delim, (size_t)(le - f));
    if (!fe) fe = le;
    while (f < fe && py_space((unsigned char)*f)) ++f;
    while (fe > f && py_space((unsigned char)fe[-1])) --fe;
    double v = 0.0;
    const bool ok = py_float(f, (size_t)(fe - f), limit, &v, buf) && std::isfinite(v);
    if (!ok) {
      if (skip_invalid) {
        ++c->skipped;
        continue;
      }
      c->err_line = lineno;
      c->err_kind = 2;
      c->err_token.assign(f, (size_t)(fe - f));
      return;
    }
    c->vals.push_back(v);
  }
}

}  // namespace

extern "C" int rqa_read_column(const char* path, char delimiter, int64_t column, int64_t offset,
                               int32_t skip_invalid, int32_t threads, double** values,
                               int64_t* count, int64_t* skipped, int64_t* err_line,
                               int64_t* err_fields, char* err, size_t errlen) {
  if (!path || !values || !count || !skipped || !err_line || !err_fields)
    return ing_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  *values = nullptr;
  *count = *skipped = *err_line = *err_fields = 0;
  if (column < 0) return ing_err(err, errlen, "column must be >= 0"), RQA_EINVAL;
  if (offset < 0) return ing_err(err, errlen, "offset must be >= 0"), RQA_EINVAL;
  if ((unsigned char)delimiter >= 0x80 || delimiter == '\n' || delimiter == '\r')
    return ing_err(err, errlen, "delimiter not supported natively"), RQA_EUNSUPPORTED;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return ing_err(err, errlen, "cannot read %s: %s", path, strerror(errno)), RQA_EIO;
  struct stat stt;
  if (fstat(fd, &stt) != 0 || S_ISDIR(stt.st_mode)) {
    close(fd);
    return ing_err(err, errlen, "cannot read %s: is a directory", path), RQA_EIO;
  }
  if (!S_ISREG(stt.st_mode)) {  // pipes, devices: the Python reader streams them
    close(fd);
    return ing_err(err, errlen, "not a regular file"), RQA_EUNSUPPORTED;
  }
  const size_t size = (size_t)stt.st_size;
  const char* data = nullptr;
  void* map = nullptr;
  if (size > 0) {
    map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (map == MAP_FAILED) {
      close(fd);
      return ing_err(err, errlen, "cannot read %s: %s", path, strerror(errno)), RQA_EIO;
    }
    data = (const char*)map;
  }
  close(fd);
  struct Unmap {
    void* m;
    size_t s;
    ~Unmap() {
      if (m && m != MAP_FAILED) munmap(m, s);
    }
  } unmap{map, size};

  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min(nt, 64));
  if (size < ((size_t)1 << 20)) nt = 1;
  // chunk boundaries just after a line terminator ("\r\n" never split)
  std::vector<Chunk> ch(nt);
  const char* end = data + size;
  const char* p = data;
  for (int t = 0; t < nt; ++t) {
    const char* q = (t == nt - 1) ? end : data + size * (size_t)(t + 1) / nt;
    if (q < p) q = p;
    while (q < end && q > data && q[-1] != '\n' && q[-1] != '\r') ++q;
    if (q < end && q > data && q[-1] == '\r' && *q == '\n') ++q;
    ch[t].b = p;
    ch[t].e = q;
    p = q;
  }
  bool ascii = true;
  {
    std::vector<std::thread> th;
    std::vector<char> ok(nt, 1);
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (const char* q = ch[t].b; q < ch[t].e; ++q)
          if ((unsigned char)*q >= 0x80) {
            ok[t] = 0;
            return;
          }
        count_lines(&ch[t]);
      });
    for (auto& x : th) x.join();
    for (int t = 0; t < nt; ++t) ascii &= ok[t] != 0;
  }
  if (!ascii) return ing_err(err, errlen, "non-ASCII content"), RQA_EUNSUPPORTED;
  int64_t line0 = 0, off = offset;
  for (int t = 0; t < nt; ++t) {
    ch[t].line0 = line0;
    ch[t].skip = std::min(off, ch[t].nonempty);
    off -= ch[t].skip;
    line0 += ch[t].lines;
  }
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] { parse_chunk(&ch[t], end, delimiter, column, skip_invalid); });
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < nt; ++t) {
    if (ch[t].err_line) {
      *err_line = ch[t].err_line;
      if (ch[t].err_kind == 1) {
        *err_fields = ch[t].err_fields;
        ing_err(err, errlen, "%s", "");
        return RQA_ECOLUMN;
      }
      // the token may hold NUL bytes: copy it raw, its length in *err_fields
      const size_t tl = std::min(ch[t].err_token.size(), errlen > 0 ? errlen - 1 : 0);
      if (errlen > 0) {
        memcpy(err, ch[t].err_token.data(), tl);
        err[tl] = '\0';
      }
      *err_fields = (int64_t)tl;
      return RQA_EPARSE;
    }
  }
  int64_t total = 0, skip_tot = 0;
  for (auto& c : ch) {
    total += (int64_t)c.vals.size();
    skip_tot += c.skipped;
  }
  *skipped = skip_tot;
  if (total == 0) return ing_err(err, errlen, "no values extracted from %s", path), RQA_EEMPTY;
  double* out = (double*)malloc((size_t)total * sizeof(double));
  if (!out) return ing_err(err, errlen, "out of host memory"), RQA_ENOMEM;
  int64_t at = 0;
  for (auto& c : ch) {
    if (!c.vals.empty()) memcpy(out + at, c.vals.data(), c.vals.size() * sizeof(double));
    at += (int64_t)c.vals.size();
  }
  *values = out;
  *count = total;
  return RQA_OK;
}

extern "C" void rqa_free(void* p) { free(p); }
