// Host-side readers for the input side of the decomposition path
// (reference formats.py:47-127).  Host memory only: no context, no GPU.
//
// * COO text (ingest_coo, formats.py:47-100): the whole file is parsed here
//   in one pass, including every rejection the reference makes.  Lines are
//   split the way Python's text mode does (universal newlines: \n, \r\n, \r)
//   and tokens the way str.split() does (ASCII whitespace incl. \x1c-\x1f);
//   integers and floats are recognised with Python's int() / float() literal
//   grammar (optional sign, '_' between digits, inf / infinity / nan for
//   floats, no hex), so a file is accepted here exactly when the reference
//   accepts it.  A rejected file returns FTT_ERR_INVALID with a
//   FttCooError (kind, 1-based line, mode, field count and the offending
//   token or line); the Python layer only formats the message.
// * MatrixMarket coordinate files (ingest_matrix_market, formats.py:103-127):
//   banner classification and a strict body reader for `real general` /
//   `real symmetric` files (symmetric entries expanded the way scipy's
//   reader orders them: stored entries in file order, then the mirrored
//   off-diagonal ones in file order).  Any body the strict reader does not
//   accept is reported as FTT_ERR_INVALID and the caller hands the file to
//   scipy.io.mmread -- the library the reference itself reads with -- for its
//   result or its exception text.
#include <errno.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "ftt_common.cuh"

namespace {

// Python str.split() / str.strip() whitespace, ASCII subset.
inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

struct Tok {
  const char *p;
  int64_t n;
};

bool read_file(const char *path, std::vector<char> &buf) {
  FILE *fh = fopen(path, "rb");
  if (!fh) return false;
  buf.clear();
  char tmp[1 << 16];
  size_t got;
  while ((got = fread(tmp, 1, sizeof tmp, fh)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  const bool bad = ferror(fh);
  fclose(fh);
  return !bad;
}

// Next line [*b, *e) under universal newlines; returns false at end of data.
bool next_line(const char *&p, const char *end, const char *&b, const char *&e) {
  if (p >= end) return false;
  b = p;
  while (p < end && *p != '\n' && *p != '\r') ++p;
  e = p;
  if (p < end) {
    if (*p == '\r' && p + 1 < end && p[1] == '\n') ++p;
    ++p;
  }
  return true;
}

void split(const char *b, const char *e, std::vector<Tok> &out) {
  out.clear();
  while (b < e) {
    while (b < e && py_space((unsigned char)*b)) ++b;
    if (b >= e) break;
    const char *s = b;
    while (b < e && !py_space((unsigned char)*b)) ++b;
    out.push_back({s, (int64_t)(b - s)});
  }
}

// Digits with single '_' separators between digits ("1_000"), at least one
// digit.  Appends the digits (underscores dropped) to `digits`.
bool py_digitpart(const char *&p, const char *e, std::string &digits) {
  if (p >= e || !is_digit(*p)) return false;
  while (p < e) {
    if (is_digit(*p)) {
      digits.push_back(*p++);
    } else if (*p == '_' && p + 1 < e && is_digit(p[1])) {
      ++p;
    } else {
      break;
    }
  }
  return true;
}

enum IntParse { INT_OK = 0, INT_BAD = 1, INT_BIG = 2 };

// Python int(token): [sign] digitpart.  INT_BIG = a valid literal whose value
// does not fit int64 (the reference then reports it out of range).
// CPython also refuses literals longer than 4300 digits (ValueError).
IntParse py_int(Tok t, int64_t *out) {
  const char *p = t.p, *e = t.p + t.n;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  std::string digits;
  if (!py_digitpart(p, e, digits) || p != e) return INT_BAD;
  if (digits.size() > 4300) return INT_BAD;
  size_t i = 0;
  while (i + 1 < digits.size() && digits[i] == '0') ++i;
  if (digits.size() - i > 19) return INT_BIG;
  unsigned long long v = 0;
  for (; i < digits.size(); ++i) v = v * 10ull + (unsigned long long)(digits[i] - '0');
  if (!neg && v > (unsigned long long)INT64_MAX) return INT_BIG;
  if (neg && v > (unsigned long long)INT64_MAX + 1ull) return INT_BIG;
  *out = neg ? (int64_t)(0ull - v) : (int64_t)v;
  return INT_OK;
}

bool ieq(const char *p, int64_t n, const char *lit) {
  const int64_t m = (int64_t)strlen(lit);
  if (n != m) return false;
  for (int64_t i = 0; i < n; ++i) {
    char c = p[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != lit[i]) return false;
  }
  return true;
}

// Python float(token): [sign] (inf | infinity | nan | decimal), decimal =
// digitpart ['.' [digitpart]] [exp] | '.' digitpart [exp], exp = (e|E) [sign]
// digitpart.  The underscore-free literal goes to strtod (correctly
// rounded, like CPython's dtoa), so the value is bit-identical.
bool py_float(Tok t, double *out) {
  const char *p = t.p, *e = t.p + t.n;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  const int64_t rest = (int64_t)(e - p);
  if (ieq(p, rest, "inf") || ieq(p, rest, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, rest, "nan")) {
    *out = neg ? -NAN : NAN;
    return true;
  }
  std::string lit;
  if (neg) lit.push_back('-');
  bool have = false;
  if (p < e && is_digit(*p)) have = py_digitpart(p, e, lit);
  if (p < e && *p == '.') {
    lit.push_back(*p++);
    if (p < e && is_digit(*p)) {
      py_digitpart(p, e, lit);
      have = true;
    }
  }
  if (!have) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    lit.push_back(*p++);
    if (p < e && (*p == '+' || *p == '-')) lit.push_back(*p++);
    if (!py_digitpart(p, e, lit)) return false;
  }
  if (p != e) return false;
  errno = 0;
  *out = strtod(lit.c_str(), nullptr);  // ERANGE: +-inf or a (sub)normal/zero, as Python
  return true;
}

char *dup_text(const char *b, int64_t n) {
  char *s = (char *)malloc((size_t)n + 1);
  if (s) {
    memcpy(s, b, (size_t)n);
    s[n] = '\0';
  }
  return s;
}

void set_err(ftt_coo_error *err, int32_t kind, int64_t line, const char *b, int64_t n) {
  err->kind = kind;
  err->line = line;
  err->text = b ? dup_text(b, n) : nullptr;
  err->text_len = b ? n : 0;
}

}  // namespace

extern "C" {

void ftt_free_host(void *p) { free(p); }

int ftt_parse_coo_text(const char *path, int32_t max_d, int32_t *d_out, int64_t *dims_out,
                       int64_t *nnz_out, int64_t **coords_out, double **vals_out,
                       ftt_coo_error *err) {
  if (!path || !d_out || !dims_out || !nnz_out || !coords_out || !vals_out || !err || max_d < 1)
    return FTT_ERR_INVALID;
  *coords_out = nullptr;
  *vals_out = nullptr;
  *nnz_out = 0;
  *d_out = 0;
  memset(err, 0, sizeof *err);
  std::vector<char> buf;
  if (!read_file(path, buf)) {
    ftt::set_error("cannot read %s", path);
    err->kind = FTT_COO_IO;
    return FTT_ERR_INVALID;
  }
  const char *p = buf.data(), *end = buf.data() + buf.size();
  // the reference opens the file as ASCII text: any other byte is a decode error
  for (size_t i = 0; i < buf.size(); ++i) {
    if ((unsigned char)buf[i] >= 0x80) {
      err->kind = FTT_COO_NONASCII;
      err->count = (int64_t)i;
      err->mode = (unsigned char)buf[i];
      return FTT_ERR_INVALID;
    }
  }
  if (buf.empty()) {
    err->kind = FTT_COO_EMPTY;
    return FTT_ERR_INVALID;
  }
  std::vector<Tok> tok;
  const char *lb, *le;
  next_line(p, end, lb, le);
  split(lb, le, tok);
  if (tok.size() < 3 || !(tok[0].n == 1 && tok[0].p[0] == '#') ||
      !(tok[1].n == 5 && memcmp(tok[1].p, "shape", 5) == 0)) {
    set_err(err, FTT_COO_HEADER, 1, nullptr, 0);
    return FTT_ERR_INVALID;
  }
  // shape extents: int() each, positive, product < 2^63 (check_shape,
  // tensor.py:47-67); the Python layer words the message from the header
  const int64_t d64 = (int64_t)tok.size() - 2;
  {
    bool ok = d64 <= max_d;
    unsigned __int128 prod = 1;
    for (int64_t k = 0; ok && k < d64; ++k) {
      int64_t v = 0;
      ok = py_int(tok[2 + k], &v) == INT_OK && v >= 1;
      if (ok) {
        prod *= (unsigned __int128)v;
        ok = prod < ((unsigned __int128)1 << 63);
        dims_out[k] = v;
      }
    }
    if (!ok) {
      set_err(err, FTT_COO_SHAPE, 1, lb, (int64_t)(le - lb));
      return FTT_ERR_INVALID;
    }
  }
  const int d = (int)d64;
  *d_out = d;
  std::vector<int64_t> coords;
  std::vector<double> vals;
  coords.reserve(buf.size() / 8);
  vals.reserve(buf.size() / (8 * (size_t)(d + 1)) + 1);
  std::vector<int64_t> idx((size_t)d);
  std::vector<IntParse> kind((size_t)d);
  int64_t line = 1;
  while (next_line(p, end, lb, le)) {
    ++line;
    split(lb, le, tok);
    if (tok.empty()) continue;
    if ((int64_t)tok.size() != d + 1) {
      set_err(err, FTT_COO_FIELDS, line, nullptr, 0);
      err->count = (int64_t)tok.size();
      return FTT_ERR_INVALID;
    }
    // all literals first (one ValueError for the entry), then ranges in
    // mode order, then finiteness -- the reference's order of checks
    bool parsed = true;
    for (int k = 0; k < d && parsed; ++k) {
      kind[k] = py_int(tok[k], &idx[k]);
      parsed = kind[k] != INT_BAD;
    }
    double v = 0.0;
    if (parsed) parsed = py_float(tok[d], &v);
    if (!parsed) {
      set_err(err, FTT_COO_UNPARSABLE, line, lb, (int64_t)(le - lb));
      return FTT_ERR_INVALID;
    }
    for (int k = 0; k < d; ++k) {
      if (kind[k] == INT_BIG || idx[k] < 1 || idx[k] > dims_out[k]) {
        set_err(err, FTT_COO_RANGE, line, tok[k].p, tok[k].n);
        err->mode = k;
        return FTT_ERR_INVALID;
      }
    }
    if (!isfinite(v)) {
      set_err(err, FTT_COO_NONFINITE, line, tok[d].p, tok[d].n);
      return FTT_ERR_INVALID;
    }
    for (int k = 0; k < d; ++k) coords.push_back(idx[k] - 1);
    vals.push_back(v);
  }
  const int64_t nnz = (int64_t)vals.size();
  int64_t *c = (int64_t *)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(nnz * d, 1));
  double *vv = (double *)malloc(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1));
  if (!c || !vv) {
    free(c);
    free(vv);
    ftt::set_error("out of host memory reading %s", path);
    return FTT_ERR_OOM;
  }
  if (nnz) {
    memcpy(c, coords.data(), sizeof(int64_t) * (size_t)(nnz * d));
    memcpy(vv, vals.data(), sizeof(double) * (size_t)nnz);
  }
  *coords_out = c;
  *vals_out = vv;
  *nnz_out = nnz;
  return FTT_OK;
}

int ftt_parse_mm_text(const char *path, int32_t *banner_out, int64_t *shape_out,
                      int64_t *nnz_out, int64_t **rows_out, int64_t **cols_out,
                      double **vals_out) {
  if (!path || !banner_out || !shape_out || !nnz_out || !rows_out || !cols_out || !vals_out)
    return FTT_ERR_INVALID;
  *rows_out = *cols_out = nullptr;
  *vals_out = nullptr;
  *nnz_out = 0;
  *banner_out = FTT_MM_NOT_MM;
  std::vector<char> buf;
  if (!read_file(path, buf)) {
    ftt::set_error("cannot read %s", path);
    return FTT_ERR_INVALID;
  }
  for (char ch : buf)
    if ((unsigned char)ch >= 0x80) return FTT_ERR_INVALID;  // the caller's text read decides
  const char *p = buf.data(), *end = buf.data() + buf.size();
  const char *lb = p, *le = p;
  std::vector<Tok> tok;
  if (next_line(p, end, lb, le)) split(lb, le, tok);
  if (tok.size() != 5 || !(tok[0].n == 14 && memcmp(tok[0].p, "%%MatrixMarket", 14) == 0)) {
    *banner_out = FTT_MM_NOT_MM;
    return FTT_OK;
  }
  bool sym = false;
  if (!ieq(tok[1].p, tok[1].n, "matrix")) {
    *banner_out = FTT_MM_OBJECT;
  } else if (!ieq(tok[2].p, tok[2].n, "coordinate")) {
    *banner_out = FTT_MM_FORMAT;
  } else if (!ieq(tok[3].p, tok[3].n, "real")) {
    *banner_out = FTT_MM_FIELD;
  } else if (ieq(tok[4].p, tok[4].n, "general") || (sym = ieq(tok[4].p, tok[4].n, "symmetric"))) {
    *banner_out = sym ? FTT_MM_SYMMETRIC : FTT_MM_GENERAL;
  } else {
    *banner_out = FTT_MM_SYMMETRY;
  }
  if (*banner_out != FTT_MM_GENERAL && *banner_out != FTT_MM_SYMMETRIC) return FTT_OK;
  // body: '%' comment lines and blank lines, "rows cols nnz", then nnz
  // entries "i j value" (1-based); anything else -> the library reader
  int64_t hdr[3] = {-1, -1, -1};
  bool have_size = false;
  std::vector<int64_t> rr, cc;
  std::vector<double> vv;
  int64_t want = 0;
  while (next_line(p, end, lb, le)) {
    split(lb, le, tok);
    if (tok.empty()) continue;
    if (tok[0].p[0] == '%') {
      if (have_size) return FTT_ERR_INVALID;
      continue;
    }
    if (!have_size) {
      if (tok.size() != 3) return FTT_ERR_INVALID;
      for (int k = 0; k < 3; ++k) {
        char *e2;
        errno = 0;
        hdr[k] = strtoll(tok[k].p, &e2, 10);
        if (errno || e2 != tok[k].p + tok[k].n || hdr[k] < 0 || !is_digit(tok[k].p[0]))
          return FTT_ERR_INVALID;
      }
      have_size = true;
      want = hdr[2];
      if (want > (int64_t)buf.size()) return FTT_ERR_INVALID;
      rr.reserve((size_t)want);
      cc.reserve((size_t)want);
      vv.reserve((size_t)want);
      continue;
    }
    if (tok.size() != 3 || (int64_t)vv.size() >= want) return FTT_ERR_INVALID;
    int64_t ij[2];
    for (int k = 0; k < 2; ++k) {
      char *e2;
      errno = 0;
      ij[k] = strtoll(tok[k].p, &e2, 10);
      if (errno || e2 != tok[k].p + tok[k].n || !is_digit(tok[k].p[0]) || ij[k] < 1 ||
          ij[k] > hdr[k])
        return FTT_ERR_INVALID;
    }
    double v;
    {
      // plain decimal literal only (digits, '.', exponent): strtod on it is
      // the value every conforming reader produces
      const char *q = tok[2].p, *e = q + tok[2].n;
      if (q < e && (*q == '+' || *q == '-')) ++q;
      bool dig = false;
      while (q < e && is_digit(*q)) { ++q; dig = true; }
      if (q < e && *q == '.') { ++q; while (q < e && is_digit(*q)) { ++q; dig = true; } }
      if (!dig) return FTT_ERR_INVALID;
      if (q < e && (*q == 'e' || *q == 'E')) {
        ++q;
        if (q < e && (*q == '+' || *q == '-')) ++q;
        if (q >= e || !is_digit(*q)) return FTT_ERR_INVALID;
        while (q < e && is_digit(*q)) ++q;
      }
      if (q != e) return FTT_ERR_INVALID;
      std::string lit(tok[2].p, (size_t)tok[2].n);
      v = strtod(lit.c_str(), nullptr);
      if (!isfinite(v)) return FTT_ERR_INVALID;
    }
    rr.push_back(ij[0] - 1);
    cc.push_back(ij[1] - 1);
    vv.push_back(v);
  }
  if (!have_size || (int64_t)vv.size() != want) return FTT_ERR_INVALID;
  if (sym) {
    if (hdr[0] != hdr[1]) return FTT_ERR_INVALID;
    const size_t n0 = vv.size();
    for (size_t i = 0; i < n0; ++i) {
      if (rr[i] != cc[i]) {
        rr.push_back(cc[i]);
        cc.push_back(rr[i]);
        vv.push_back(vv[i]);
      }
    }
  }
  const int64_t n = (int64_t)vv.size();
  int64_t *r = (int64_t *)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(n, 1));
  int64_t *c = (int64_t *)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(n, 1));
  double *w = (double *)malloc(sizeof(double) * (size_t)std::max<int64_t>(n, 1));
  if (!r || !c || !w) {
    free(r);
    free(c);
    free(w);
    ftt::set_error("out of host memory reading %s", path);
    return FTT_ERR_OOM;
  }
  if (n) {
    memcpy(r, rr.data(), sizeof(int64_t) * (size_t)n);
    memcpy(c, cc.data(), sizeof(int64_t) * (size_t)n);
    memcpy(w, vv.data(), sizeof(double) * (size_t)n);
  }
  shape_out[0] = hdr[0];
  shape_out[1] = hdr[1];
  *rows_out = r;
  *cols_out = c;
  *vals_out = w;
  *nnz_out = n;
  return FTT_OK;
}

}  // extern "C"
