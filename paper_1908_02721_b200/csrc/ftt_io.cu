// Host-side COO text reader (formats.py:47-100 of the reference, whose
// ingest_coo is a per-line Python loop): one pass over the file with
// strtoll / strtod into malloc'd arrays.  Only the fast path lives here: on
// the first malformed line the reader stops and reports the line number;
// the Python mirror then re-reads that file with the reference's loop to
// raise the reference's exact FormatError text.
#include <errno.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "ftt_common.cuh"

namespace {

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

}  // namespace

extern "C" {

void ftt_free_host(void *p) { free(p); }

// Returns FTT_OK with the canonical-input arrays (1-based indices already
// shifted to 0-based) or FTT_ERR_INVALID with *bad_line = the first line the
// fast path rejects (1 = header, 0 = empty file / I/O error).
int ftt_parse_coo_text(const char *path, int32_t *d_out, int64_t *dims_out, int64_t *nnz_out,
                       int64_t **coords_out, double **vals_out, int64_t *bad_line) {
  if (!path || !d_out || !dims_out || !nnz_out || !coords_out || !vals_out || !bad_line)
    return FTT_ERR_INVALID;
  *coords_out = nullptr;
  *vals_out = nullptr;
  *nnz_out = 0;
  *bad_line = 0;
  FILE *fh = fopen(path, "rb");
  if (!fh) {
    ftt::set_error("cannot open %s", path);
    return FTT_ERR_INVALID;
  }
  fseek(fh, 0, SEEK_END);
  const long size = ftell(fh);
  fseek(fh, 0, SEEK_SET);
  std::vector<char> buf((size_t)(size > 0 ? size : 0) + 1);
  const size_t got = size > 0 ? fread(buf.data(), 1, (size_t)size, fh) : 0;
  fclose(fh);
  buf[got] = '\0';
  if (got == 0) return FTT_ERR_INVALID;  // empty file: the Python path words the error
  char *p = buf.data(), *end = buf.data() + got;
  // header: "# shape n1 ... nd"
  char *eol = (char *)memchr(p, '\n', end - p);
  if (!eol) eol = end;
  *eol = '\0';
  *bad_line = 1;
  {
    char *q = p;
    while (q < eol && is_space(*q)) ++q;
    if (*q != '#') return FTT_ERR_INVALID;
    ++q;
    if (!is_space(*q)) return FTT_ERR_INVALID;
    while (q < eol && is_space(*q)) ++q;
    if (strncmp(q, "shape", 5) != 0 || !is_space(q[5])) return FTT_ERR_INVALID;
    q += 5;
    int d = 0;
    while (true) {
      while (q < eol && is_space(*q)) ++q;
      if (q >= eol || !*q) break;
      char *e2;
      errno = 0;
      const long long v = strtoll(q, &e2, 10);
      if (e2 == q || errno || (e2 < eol && *e2 && !is_space(*e2)) || v < 1 || d >= 32)
        return FTT_ERR_INVALID;
      dims_out[d++] = v;
      q = e2;
    }
    if (d < 1) return FTT_ERR_INVALID;
    *d_out = d;
  }
  const int d = *d_out;
  std::vector<int64_t> coords;
  std::vector<double> vals;
  coords.reserve((size_t)got / 8);
  vals.reserve((size_t)got / (8 * (d + 1)) + 1);
  int64_t line = 1;
  p = eol + 1;
  while (p < end) {
    ++line;
    char *le = (char *)memchr(p, '\n', end - p);
    if (!le) le = end;
    *le = '\0';
    char *q = p;
    while (q < le && is_space(*q)) ++q;
    if (q < le && *q) {
      for (int k = 0; k < d; ++k) {
        while (q < le && is_space(*q)) ++q;
        char *e2;
        errno = 0;
        const long long v = strtoll(q, &e2, 10);
        if (e2 == q || errno || (e2 < le && *e2 && !is_space(*e2)) || v < 1 || v > dims_out[k]) {
          *bad_line = line;
          return FTT_ERR_INVALID;
        }
        coords.push_back(v - 1);
        q = e2;
      }
      while (q < le && is_space(*q)) ++q;
      // plain decimal floats only (hex floats, which strtod accepts and
      // Python's float() does not, go to the reference loop)
      if (q[0] == '0' && (q[1] == 'x' || q[1] == 'X')) {
        *bad_line = line;
        return FTT_ERR_INVALID;
      }
      char *e2;
      errno = 0;
      const double v = strtod(q, &e2);
      if (e2 == q || (e2 < le && *e2 && !is_space(*e2)) || !isfinite(v)) {
        *bad_line = line;
        return FTT_ERR_INVALID;
      }
      q = e2;
      while (q < le && is_space(*q)) ++q;
      if (q < le && *q) {  // extra fields
        *bad_line = line;
        return FTT_ERR_INVALID;
      }
      vals.push_back(v);
    }
    p = le + 1;
  }
  const int64_t nnz = (int64_t)vals.size();
  int64_t *c = (int64_t *)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(nnz * d, 1));
  double *v = (double *)malloc(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1));
  if (!c || !v) {
    free(c);
    free(v);
    ftt::set_error("out of host memory reading %s", path);
    return FTT_ERR_OOM;
  }
  if (nnz) {
    memcpy(c, coords.data(), sizeof(int64_t) * (size_t)(nnz * d));
    memcpy(v, vals.data(), sizeof(double) * (size_t)nnz);
  }
  *coords_out = c;
  *vals_out = v;
  *nnz_out = nnz;
  *bad_line = 0;
  return FTT_OK;
}

}  // extern "C"
