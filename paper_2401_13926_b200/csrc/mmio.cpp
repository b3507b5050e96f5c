// Matrix Market ingestion in C++ (mmio.load_matrix_market / load_vector, mmio.py:36-130;
// SURVEY.md §8f row 4): the reference parses the sequence files line by line in Python,
// which dominates wall time for the 10M-line ACTIVSg70k-sized files.  Same accepted
// dialect and the same errors (with the offending line number): `matrix coordinate real
// general|symmetric` (symmetric: lower triangle only, 1-based indices) and `matrix array real
// general` n x 1 vectors.  Values go through strtod (correctly rounded, like Python float()).
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kkt_internal.h"

namespace kkt {

namespace {

struct MMFile {
  std::string path, data;
  std::vector<size_t> line_start;  // offsets of every line
  bool ok = false;
};

int mm_error(const std::string &path, long line, const std::string &msg) {
  return set_error(KKT_ERR_BAD_ARG, path + ":" + std::to_string(line) + ": " + msg);
}

int slurp(const char *path, MMFile &f) {
  f.path = path;
  FILE *fp = std::fopen(path, "rb");
  if (!fp) return set_error(KKT_ERR_BAD_ARG, std::string(path) + ": cannot open: " + std::strerror(errno));
  std::fseek(fp, 0, SEEK_END);
  const long sz = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  f.data.resize(sz > 0 ? (size_t)sz : 0);
  if (sz > 0 && std::fread(&f.data[0], 1, (size_t)sz, fp) != (size_t)sz) {
    std::fclose(fp);
    return set_error(KKT_ERR_BAD_ARG, std::string(path) + ": read error");
  }
  std::fclose(fp);
  size_t p = 0;
  while (p < f.data.size()) {
    f.line_start.push_back(p);
    const void *nl = std::memchr(f.data.data() + p, '\n', f.data.size() - p);
    if (!nl) break;
    p = (size_t)((const char *)nl - f.data.data()) + 1;
  }
  return KKT_OK;
}

// [b, e) of line i without the trailing newline / carriage return
void line_span(const MMFile &f, size_t i, const char *&b, const char *&e) {
  b = f.data.data() + f.line_start[i];
  e = (i + 1 < f.line_start.size()) ? f.data.data() + f.line_start[i + 1] : f.data.data() + f.data.size();
  while (e > b && (e[-1] == '\n' || e[-1] == '\r')) --e;
}

void tokens(const char *b, const char *e, std::vector<std::string> &out) {
  out.clear();
  while (b < e) {
    while (b < e && (*b == ' ' || *b == '\t' || *b == '\r' || *b == '\v' || *b == '\f')) ++b;
    const char *s = b;
    while (b < e && !(*b == ' ' || *b == '\t' || *b == '\r' || *b == '\v' || *b == '\f')) ++b;
    if (b > s) out.emplace_back(s, b);
  }
}

bool blank_or_comment(const char *b, const char *e) {
  while (b < e && (*b == ' ' || *b == '\t' || *b == '\r')) ++b;
  return b == e || *b == '%';
}

std::string lower(std::string s) {
  for (char &c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

bool parse_i64(const std::string &s, int64_t &v) {
  char *end = nullptr;
  errno = 0;
  const long long x = std::strtoll(s.c_str(), &end, 10);
  if (errno || end == s.c_str() || *end) return false;
  v = (int64_t)x;
  return true;
}

bool parse_f64(const std::string &s, double &v) {
  char *end = nullptr;
  errno = 0;
  v = std::strtod(s.c_str(), &end);
  return end != s.c_str() && !*end && errno != EINVAL;
}

// header + size line; fmt 0 coordinate / 1 array, sym 0 general / 1 symmetric
int header(const MMFile &f, int &fmt, int &sym, size_t &size_line) {
  if (f.line_start.empty()) return mm_error(f.path, 1, "empty file");
  const char *b, *e;
  line_span(f, 0, b, e);
  std::vector<std::string> t;
  tokens(b, e, t);
  if (t.size() < 4 || t[0] != "%%MatrixMarket" || lower(t[1]) != "matrix")
    return mm_error(f.path, 1, "not a Matrix Market matrix header");
  const std::string fm = lower(t[2]), fld = lower(t[3]), sy = t.size() > 4 ? lower(t[4]) : "general";
  if (fld != "real") return mm_error(f.path, 1, "only the 'real' field is supported, got '" + fld + "'");
  if (fm != "coordinate" && fm != "array") return mm_error(f.path, 1, "unsupported format '" + fm + "'");
  if (sy != "general" && sy != "symmetric") return mm_error(f.path, 1, "unsupported symmetry '" + sy + "'");
  fmt = fm == "coordinate" ? 0 : 1;
  sym = sy == "symmetric" ? 1 : 0;
  size_t ln = 1;
  while (ln < f.line_start.size()) {
    line_span(f, ln, b, e);
    if (!blank_or_comment(b, e)) break;
    ++ln;
  }
  if (ln >= f.line_start.size()) return mm_error(f.path, (long)ln + 1, "missing size line");
  size_line = ln;
  return KKT_OK;
}

}  // namespace

// info[0..4] = {format (0 coordinate, 1 array), symmetric, rows, cols, nnz (array: rows)}
static int sizes(const MMFile &f, int fmt, int sym, size_t ln, int64_t *info) {
  const char *b, *e;
  line_span(f, ln, b, e);
  std::vector<std::string> t;
  tokens(b, e, t);
  int64_t r = 0, c = 0, z = 0;
  if (fmt == 0) {
    if (t.size() != 3) return mm_error(f.path, (long)ln + 1, "size line must be 'rows cols nnz'");
    if (!parse_i64(t[0], r) || !parse_i64(t[1], c) || !parse_i64(t[2], z))
      return mm_error(f.path, (long)ln + 1, "bad size line");
  } else {
    if (t.size() != 2) return mm_error(f.path, (long)ln + 1, "array size line must be 'rows cols'");
    if (!parse_i64(t[0], r) || !parse_i64(t[1], c)) return mm_error(f.path, (long)ln + 1, "bad size line");
    z = r;
  }
  info[0] = fmt;
  info[1] = sym;
  info[2] = r;
  info[3] = c;
  info[4] = z;
  return KKT_OK;
}

int mm_info(const char *path, int64_t *info) {
  MMFile f;
  int rc = slurp(path, f);
  if (rc) return rc;
  int fmt = 0, sym = 0;
  size_t ln = 0;
  if ((rc = header(f, fmt, sym, ln))) return rc;
  return sizes(f, fmt, sym, ln, info);
}

// coordinate entries, 0-based (rows/cols) in file order; checks as mmio.py:66-91
int mm_read_coo(const char *path, int64_t nnz, int64_t *rows, int64_t *cols, double *vals) {
  MMFile f;
  int rc = slurp(path, f);
  if (rc) return rc;
  int fmt = 0, sym = 0;
  size_t ln = 0;
  if ((rc = header(f, fmt, sym, ln))) return rc;
  if (fmt != 0) return mm_error(f.path, 1, "expected a coordinate matrix, got 'array'");
  int64_t info[5];
  if ((rc = sizes(f, fmt, sym, ln, info))) return rc;
  const int64_t n_rows = info[2], n_cols = info[3];
  if (info[4] != nnz) return set_error(KKT_ERR_BAD_ARG, "mm_read_coo: nnz disagrees with the file");
  int64_t k = 0;
  std::vector<std::string> t;
  for (size_t i = ln + 1; i < f.line_start.size(); ++i) {
    const char *b, *e;
    line_span(f, i, b, e);
    if (blank_or_comment(b, e)) continue;
    if (k >= nnz) return mm_error(f.path, (long)i + 1, "more entries than the declared " + std::to_string(nnz));
    tokens(b, e, t);
    if (t.size() != 3) return mm_error(f.path, (long)i + 1, "expected 'row col value'");
    int64_t r = 0, c = 0;
    double v = 0.0;
    if (!parse_i64(t[0], r) || !parse_i64(t[1], c) || !parse_f64(t[2], v))
      return mm_error(f.path, (long)i + 1, "cannot parse entry");
    if (!(1 <= r && r <= n_rows && 1 <= c && c <= n_cols))
      return mm_error(f.path, (long)i + 1, "index (" + std::to_string(r) + ", " + std::to_string(c) +
                                               ") out of range for a " + std::to_string(n_rows) + "x" +
                                               std::to_string(n_cols) + " matrix");
    if (sym && c > r) return mm_error(f.path, (long)i + 1, "symmetric file lists entry above the diagonal");
    rows[k] = r - 1;
    cols[k] = c - 1;
    vals[k] = v;
    ++k;
  }
  if (k != nnz)
    return set_error(KKT_ERR_BAD_ARG, f.path + ": declared " + std::to_string(nnz) + " entries but found " +
                                          std::to_string(k));
  return KKT_OK;
}

// array n x 1 values (mmio.py:116-130)
int mm_read_array(const char *path, int64_t n, double *out) {
  MMFile f;
  int rc = slurp(path, f);
  if (rc) return rc;
  int fmt = 0, sym = 0;
  size_t ln = 0;
  if ((rc = header(f, fmt, sym, ln))) return rc;
  if (fmt != 1) return mm_error(f.path, 1, "expected an array vector");
  int64_t info[5];
  if ((rc = sizes(f, fmt, sym, ln, info))) return rc;
  if (info[3] != 1) return mm_error(f.path, (long)ln + 1, "expected a single-column vector");
  if (info[2] != n) return set_error(KKT_ERR_BAD_ARG, "mm_read_array: length disagrees with the file");
  int64_t k = 0;
  std::vector<std::string> t;
  for (size_t i = ln + 1; i < f.line_start.size(); ++i) {
    const char *b, *e;
    line_span(f, i, b, e);
    if (blank_or_comment(b, e)) continue;
    if (k >= n) return mm_error(f.path, (long)i + 1, "more entries than declared");
    tokens(b, e, t);
    double v = 0.0;
    if (t.size() != 1 || !parse_f64(t[0], v)) return mm_error(f.path, (long)i + 1, "cannot parse value");
    out[k++] = v;
  }
  if (k != n)
    return set_error(KKT_ERR_BAD_ARG, f.path + ": declared " + std::to_string(n) + " values but found " +
                                          std::to_string(k));
  return KKT_OK;
}

}  // namespace kkt

extern "C" {
int kkt_mm_info(const char *path, int64_t *info) {
  if (!path || !info) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  return kkt::mm_info(path, info);
}
int kkt_mm_read_coo(const char *path, int64_t nnz, int64_t *rows, int64_t *cols, double *vals) {
  if (!path || (nnz > 0 && (!rows || !cols || !vals))) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  return kkt::mm_read_coo(path, nnz, rows, cols, vals);
}
int kkt_mm_read_array(const char *path, int64_t n, double *out) {
  if (!path || (n > 0 && !out)) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  return kkt::mm_read_array(path, n, out);
}
}
