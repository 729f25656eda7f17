// Matrix Market text I/O for graphs, factors, vectors and permutations
// (SURVEY §8(f)-4). Same files, byte for byte, as the reference:
//   read_matrix_market / read_laplacian   proj/src/matrix_market.cpp:65-135
//   validate_laplacian                    proj/src/graph.cpp:99-186
//   write_matrix_market                   proj/src/matrix_market.cpp:137-159
//   write_factor / read_factor            proj/src/matrix_market.cpp:161-266
//   write_vector / read_vector            proj/src/matrix_market.cpp:268-304
//   ordering_from_file / write_permutation proj/src/ordering.cpp:72-93
// Values are written as %.17g (exact binary64 round trip). The reference
// formats and parses one line at a time through stdio / iostreams; here the
// text is formatted with std::to_chars (specified to match printf "%.17g") and
// parsed with std::from_chars (correctly rounded, like strtod) by all host
// threads over newline-aligned chunks, then assembled in file order -- the
// factor files of the BASELINE configs are 22M-266M lines.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../../include/parac_gpu.h"
#include "errors.hpp"
#include "graph_build.hpp"

namespace parac_gpu {
namespace {

int host_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(1u, std::min(hw, 64u)));
}

// Runs f(t, lo, hi) over [0, n) split into at most `parts` contiguous ranges.
template <typename F>
void split_run(std::int64_t n, int parts, F&& f) {
  parts = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(parts, n)));
  if (parts <= 1) {
    f(0, std::int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < parts; ++t) {
    const std::int64_t lo = n * t / parts, hi = n * (t + 1) / parts;
    pool.emplace_back([&f, t, lo, hi] { f(t, lo, hi); });
  }
  for (auto& th : pool) th.join();
}

[[noreturn]] void parse_fail(const std::string& path, long line, const std::string& what) {
  throw Failure{parse_error, path + ":" + std::to_string(line) + ": " + what};
}

std::string slurp(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw Failure{io_error, "cannot open " + path};
  std::string s;
  char buf[1 << 16];
  std::size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) s.append(buf, got);
  std::fclose(f);
  return s;
}

// std::getline over an in-memory buffer (LineReader, matrix_market.cpp:29-45)
struct Lines {
  std::string_view text;
  std::size_t pos = 0;
  long line_no = 0;
  bool next(std::string_view& out) {
    if (pos >= text.size()) return false;
    const std::size_t e = text.find('\n', pos);
    const std::size_t stop = e == std::string_view::npos ? text.size() : e;
    out = text.substr(pos, stop - pos);
    pos = e == std::string_view::npos ? text.size() : e + 1;
    ++line_no;
    return true;
  }
};

bool blank(std::string_view l) { return l.find_first_not_of(" \t\r") == std::string_view::npos; }

// istream-style token parsing: skip whitespace, optional '+', then from_chars.
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }
inline const char* skip_ws(const char* p, const char* e) {
  while (p < e && is_ws(*p)) ++p;
  return p;
}
bool read_ll(const char*& p, const char* e, long long& v) {
  p = skip_ws(p, e);
  if (p < e && *p == '+') ++p;
  const auto r = std::from_chars(p, e, v);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}
bool read_double(const char*& p, const char* e, double& v) {
  p = skip_ws(p, e);
  const char* q = p;
  if (q < e && *q == '+') ++q;
  // iostreams do not accept inf / nan spellings
  const char* d = q < e && *q == '-' ? q + 1 : q;
  if (d < e && (*d == 'i' || *d == 'I' || *d == 'n' || *d == 'N')) return false;
  const auto r = std::from_chars(q, e, v, std::chars_format::general);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

std::vector<std::string> header_words(std::string_view l) {
  std::vector<std::string> w;
  const char* p = l.data();
  const char* e = p + l.size();
  while (true) {
    p = skip_ws(p, e);
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws(*p)) ++p;
    w.emplace_back(s, p);
  }
  return w;
}

struct Triplet {
  std::int32_t row, col;
  double value;
};

// Parse the data lines of [text, end) in parallel: every line that is not a
// comment (first char '%', when skip_comment) nor blank (when skip_blank) is
// one record of `fields` values; keeps the first `want` records in file order.
// rec(line, p, e, out) parses one record or returns an error message.
template <typename R, typename Parse>
std::vector<R> parse_records(const std::string& path, std::string_view text, long first_line, std::int64_t want,
                             bool skip_blank, Parse&& rec, const char* eof_msg) {
  const int T = text.size() > (1u << 20) ? host_threads() : 1;
  // newline-aligned chunk starts
  std::vector<std::size_t> start(static_cast<std::size_t>(T) + 1, text.size());
  start[0] = 0;
  for (int t = 1; t < T; ++t) {
    std::size_t s = text.size() * static_cast<std::size_t>(t) / static_cast<std::size_t>(T);
    s = text.find('\n', std::max(s, start[t - 1]));
    start[t] = s == std::string_view::npos ? text.size() : s + 1;
  }
  struct Part {
    std::vector<R> out;
    long lines = 0;
    long err_line = -1;  // chunk-local line of the first error
    std::string err;
  };
  std::vector<Part> parts(static_cast<std::size_t>(T));
  split_run(T, T, [&](int, std::int64_t lo, std::int64_t hi) {
    for (std::int64_t t = lo; t < hi; ++t) {
      Part& P = parts[static_cast<std::size_t>(t)];
      Lines L{text.substr(start[t], start[t + 1] - start[t])};
      std::string_view line;
      while (L.next(line)) {
        if (!line.empty() && line[0] == '%') continue;
        if (skip_blank && blank(line)) continue;
        R r;
        const char* err = rec(line.data(), line.data() + line.size(), r);
        if (err) {
          P.err_line = L.line_no;
          P.err = err;
          break;
        }
        P.out.push_back(r);
      }
      P.lines = L.line_no;
    }
  });
  std::vector<R> out;
  out.reserve(static_cast<std::size_t>(std::max<std::int64_t>(want, 0)));
  long line_base = first_line;
  for (int t = 0; t < T && static_cast<std::int64_t>(out.size()) < want; ++t) {
    Part& P = parts[static_cast<std::size_t>(t)];
    const std::size_t take = std::min<std::size_t>(P.out.size(), static_cast<std::size_t>(want) - out.size());
    out.insert(out.end(), P.out.begin(), P.out.begin() + static_cast<std::ptrdiff_t>(take));
    if (static_cast<std::int64_t>(out.size()) < want && P.err_line >= 0) parse_fail(path, line_base + P.err_line, P.err);
    // a chunk that stopped at an error has not counted its later lines
    line_base += P.err_line >= 0 ? P.err_line : P.lines;
  }
  if (static_cast<std::int64_t>(out.size()) < want) parse_fail(path, line_base, eof_msg);
  return out;
}

// ---- formatting -------------------------------------------------------------
struct Out {
  std::string s;
  void i(long long v) {
    char b[24];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    s.append(b, r.ptr);
  }
  void d(double v) {  // printf("%.17g")
    char b[40];
    const auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::general, 17);
    s.append(b, r.ptr);
  }
  void c(char ch) { s.push_back(ch); }
  void str(const char* t) { s.append(t); }
};

struct File {
  std::FILE* f = nullptr;
  explicit File(const std::string& path, const char* what = "cannot write ") : f(std::fopen(path.c_str(), "wb")) {
    if (!f) throw Failure{io_error, what + path};
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void put(const std::string& s) {
    if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) throw Failure{io_error, "short write"};
  }
};

// Format items [0, n) in parallel ranges balanced by `weight` prefix (or by
// count) and write them in order.
template <typename Fmt>
void write_parallel(File& f, std::int64_t n, const std::int64_t* prefix, Fmt&& fmt) {
  const int T = n > 65536 ? host_threads() : 1;
  std::vector<std::int64_t> cut(static_cast<std::size_t>(T) + 1, n);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    if (prefix) {
      const std::int64_t target = prefix[n] / T * t;
      cut[t] = std::max(cut[t - 1], static_cast<std::int64_t>(std::lower_bound(prefix, prefix + n, target) - prefix));
    } else {
      cut[t] = n * t / T;
    }
  }
  std::vector<Out> outs(static_cast<std::size_t>(T));
  split_run(T, T, [&](int, std::int64_t lo, std::int64_t hi) {
    for (std::int64_t t = lo; t < hi; ++t)
      for (std::int64_t k = cut[t]; k < cut[t + 1]; ++k) fmt(outs[static_cast<std::size_t>(t)], k);
  });
  for (auto& o : outs) f.put(o.s);
}

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<std::size_t>(v.size(), 1)));
  if (!p) throw Failure{internal_error, "out of host memory"};
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

// validate_laplacian, proj/src/graph.cpp:99-186 (sequential: the duplicate
// merge sums in std::sort's order, reproduced by sorting the same sequence)
void validate_laplacian(std::int32_t n, const std::vector<Triplet>& triplets, parac_graph* out) {
  std::vector<Triplet> off;
  std::vector<double> diag(static_cast<std::size_t>(n), 0.0), row_abs(static_cast<std::size_t>(n), 0.0),
      row_sum(static_cast<std::size_t>(n), 0.0);
  for (const Triplet& t : triplets) {
    if (t.row < 0 || t.col < 0 || t.row >= n || t.col >= n)
      throw Failure{parse_error,
                    "index out of range: (" + std::to_string(t.row) + ", " + std::to_string(t.col) + ")"};
    if (t.value == 0.0) continue;
    if (t.row == t.col)
      diag[static_cast<std::size_t>(t.row)] += t.value;
    else
      off.push_back(t);
  }
  auto less = [](const Triplet& a, const Triplet& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; };
  std::sort(off.begin(), off.end(), less);
  std::vector<Triplet> merged;
  merged.reserve(off.size());
  for (const Triplet& t : off) {
    if (!merged.empty() && merged.back().row == t.row && merged.back().col == t.col)
      merged.back().value += t.value;
    else
      merged.push_back(t);
  }
  for (const Triplet& t : merged) {
    const Triplet probe{t.col, t.row, 0.0};
    const auto it = std::lower_bound(merged.begin(), merged.end(), probe, less);
    const Triplet* mirror = (it == merged.end() || it->row != t.col || it->col != t.row) ? nullptr : &*it;
    const double scale = std::max(std::abs(t.value), mirror ? std::abs(mirror->value) : 0.0);
    if (mirror == nullptr || std::abs(mirror->value - t.value) > 1e-12 * scale)
      throw Failure{asymmetric_input, "row " + std::to_string(t.row) + " entry (" + std::to_string(t.row) + ", " +
                                          std::to_string(t.col) + ") has no symmetric match"};
    if (t.value > 0.0)
      throw Failure{positive_off_diagonal, "row " + std::to_string(t.row) + " off-diagonal (" +
                                               std::to_string(t.row) + ", " + std::to_string(t.col) +
                                               ") = " + std::to_string(t.value)};
  }
  for (std::int32_t v = 0; v < n; ++v) {
    row_sum[static_cast<std::size_t>(v)] = diag[static_cast<std::size_t>(v)];
    row_abs[static_cast<std::size_t>(v)] = std::abs(diag[static_cast<std::size_t>(v)]);
  }
  for (const Triplet& t : merged) {
    row_sum[static_cast<std::size_t>(t.row)] += t.value;
    row_abs[static_cast<std::size_t>(t.row)] += std::abs(t.value);
  }
  for (std::int32_t v = 0; v < n; ++v) {
    const std::size_t i = static_cast<std::size_t>(v);
    if (std::abs(row_sum[i]) > 1e-10 * row_abs[i])
      throw Failure{row_sum_violation, "row " + std::to_string(v) + " sums to " + std::to_string(row_sum[i])};
  }
  std::vector<Edge> edges;
  edges.reserve(merged.size() / 2);
  for (const Triplet& t : merged)
    if (t.row < t.col) edges.push_back({t.row, t.col, -t.value});
  build_graph(n, edges, out);
}

std::vector<std::int32_t> read_positions(const std::string& path, std::int32_t n) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw Failure{io_error, "cannot open permutation file " + path};
  std::fclose(f);
  const std::string text = slurp(path);
  std::vector<std::int32_t> pos;
  pos.reserve(static_cast<std::size_t>(std::max(n, 0)));
  const char* p = text.data();
  const char* e = p + text.size();
  long long v;
  while (read_ll(p, e, v)) pos.push_back(static_cast<std::int32_t>(v));
  if (static_cast<std::int32_t>(pos.size()) != n)
    throw Failure{not_a_permutation,
                  "expected " + std::to_string(n) + " entries, found " + std::to_string(pos.size())};
  std::vector<std::int32_t> inv(static_cast<std::size_t>(n), -1);
  for (std::int32_t v2 = 0; v2 < n; ++v2) {  // Ordering::from_positions, src/ordering.cpp:22-36
    const std::int32_t q = pos[static_cast<std::size_t>(v2)];
    if (q < 0 || q >= n || inv[static_cast<std::size_t>(q)] != -1)
      throw Failure{not_a_permutation, "position " + std::to_string(q) + " for vertex " + std::to_string(v2)};
    inv[static_cast<std::size_t>(q)] = v2;
  }
  return pos;
}

}  // namespace
}  // namespace parac_gpu

using namespace parac_gpu;

extern "C" {

int parac_read_laplacian(const char* path_c, parac_graph* out) {
  return guarded([&] {
    const std::string path(path_c ? path_c : "");
    const std::string text = slurp(path);
    Lines L{text};
    std::string_view line;
    if (!L.next(line)) parse_fail(path, L.line_no, "empty file");
    const auto w = header_words(line);
    if (w.empty() || w[0] != "%%MatrixMarket") parse_fail(path, L.line_no, "missing banner");
    const std::string object = w.size() > 1 ? lower(w[1]) : "", format = w.size() > 2 ? lower(w[2]) : "",
                      field = w.size() > 3 ? lower(w[3]) : "", symmetry = w.size() > 4 ? lower(w[4]) : "";
    if (object != "matrix" || format != "coordinate" || field != "real" ||
        (symmetry != "symmetric" && symmetry != "general"))
      throw Failure{unsupported_field, path + ": matrix coordinate real {symmetric|general} required, got \"" +
                                           object + " " + format + " " + field + " " + symmetry + "\""};
    long long rows = 0, cols = 0, nnz = 0;
    bool have = false;
    while (L.next(line)) {
      if (!line.empty() && line[0] == '%') continue;
      if (blank(line)) continue;
      const char* p = line.data();
      const char* e = p + line.size();
      if (!(read_ll(p, e, rows) && read_ll(p, e, cols) && read_ll(p, e, nnz)))
        parse_fail(path, L.line_no, "malformed size line");
      have = true;
      break;
    }
    if (!have) parse_fail(path, L.line_no, "missing size line");
    const bool symmetric = symmetry == "symmetric";
    struct Rec {
      long long i, j;
      double v;
    };
    auto rec = [&](const char* p, const char* e, Rec& r) -> const char* {
      if (!(read_ll(p, e, r.i) && read_ll(p, e, r.j) && read_double(p, e, r.v))) return "malformed entry";
      if (r.i < 1 || r.j < 1 || r.i > rows || r.j > cols) return "index out of bounds";
      return nullptr;
    };
    const std::vector<Rec> recs = parse_records<Rec>(path, std::string_view(text).substr(L.pos), L.line_no, nnz,
                                                     true, rec, "unexpected end of file");
    if (rows != cols) throw Failure{parse_error, path + ": matrix is not square"};
    std::vector<Triplet> trip;
    trip.reserve(recs.size() * (symmetric ? 2 : 1));
    for (const Rec& r : recs) {
      const Triplet t{static_cast<std::int32_t>(r.i - 1), static_cast<std::int32_t>(r.j - 1), r.v};
      trip.push_back(t);
      if (symmetric && t.row != t.col) trip.push_back({t.col, t.row, t.value});
    }
    validate_laplacian(static_cast<std::int32_t>(rows), trip, out);
  });
}

int parac_write_matrix_market(const char* path, const parac_csr* g) {
  return guarded([&] {
    if (!g || g->n < 0) throw Failure{dimension_mismatch, "bad graph"};
    const std::int32_t n = g->n;
    // nnz_lower + n entries; wdeg summed left to right in neighbour order
    std::vector<std::int64_t> lines(static_cast<std::size_t>(n) + 1, 0);
    for (std::int32_t v = 0; v < n; ++v) {
      std::int64_t lo = 0;
      for (std::int64_t p = g->ptr[v]; p < g->ptr[v + 1]; ++p) lo += g->adj[p] < v;
      lines[static_cast<std::size_t>(v) + 1] = lines[static_cast<std::size_t>(v)] + 1 + lo;
    }
    File f(path);
    Out h;
    h.str("%%MatrixMarket matrix coordinate real symmetric\n");
    h.i(n);
    h.c(' ');
    h.i(n);
    h.c(' ');
    h.i(lines[static_cast<std::size_t>(n)]);
    h.c('\n');
    f.put(h.s);
    write_parallel(f, n, lines.data(), [&](Out& o, std::int64_t v) {
      double wd = 0.0;
      for (std::int64_t p = g->ptr[v]; p < g->ptr[v + 1]; ++p) wd += g->w[p];
      o.i(v + 1);
      o.c(' ');
      o.i(v + 1);
      o.c(' ');
      o.d(wd);
      o.c('\n');
      for (std::int64_t p = g->ptr[v]; p < g->ptr[v + 1]; ++p)
        if (g->adj[p] < v) {
          o.i(v + 1);
          o.c(' ');
          o.i(g->adj[p] + 1);
          o.c(' ');
          o.d(-g->w[p]);
          o.c('\n');
        }
    });
  });
}

int parac_write_factor(const char* stem_c, int32_t n, const int64_t* col_ptr, const int32_t* rows,
                       const double* values, const double* diag) {
  return guarded([&] {
    if (n < 0 || !col_ptr) throw Failure{dimension_mismatch, "bad factor"};
    const std::string stem(stem_c ? stem_c : "");
    {
      File f(stem + ".G.mtx");
      Out h;
      h.str("%%MatrixMarket matrix coordinate real general\n");
      h.i(n);
      h.c(' ');
      h.i(n);
      h.c(' ');
      h.i(col_ptr[n]);
      h.c('\n');
      f.put(h.s);
      write_parallel(f, n, col_ptr, [&](Out& o, std::int64_t k) {
        for (std::int64_t p = col_ptr[k]; p < col_ptr[k + 1]; ++p) {
          o.i(rows[p] + 1);
          o.c(' ');
          o.i(k + 1);
          o.c(' ');
          o.d(values[p]);
          o.c('\n');
        }
      });
    }
    {
      File f(stem + ".D.mtx");
      Out h;
      h.str("%%MatrixMarket matrix array real general\n");
      h.i(n);
      h.str(" 1\n");
      f.put(h.s);
      write_parallel(f, n, nullptr, [&](Out& o, std::int64_t k) {
        o.d(diag[k]);
        o.c('\n');
      });
    }
  });
}

void parac_factor_free(parac_factor* f) {
  if (!f) return;
  std::free(f->col_ptr);
  std::free(f->rows);
  std::free(f->values);
  std::free(f->diag);
  std::free(f->perm);
  std::memset(f, 0, sizeof(*f));
}

int parac_read_factor(const char* stem_c, const char* perm_path, parac_factor* out) {
  return guarded([&] {
    const std::string stem(stem_c ? stem_c : "");
    std::memset(out, 0, sizeof(*out));
    std::int32_t n = 0;
    std::vector<std::int64_t> col_ptr;
    std::vector<std::int32_t> rows_out;
    std::vector<double> vals_out;
    {
      const std::string path = stem + ".G.mtx";
      const std::string text = slurp(path);
      Lines L{text};
      std::string_view line;
      if (!L.next(line)) parse_fail(path, L.line_no, "empty file");
      if (line.rfind("%%MatrixMarket matrix coordinate real general", 0) != 0)
        throw Failure{unsupported_field, path + ": expected coordinate real general"};
      long long rows = 0, cols = 0, nnz = 0;
      while (L.next(line)) {
        if (!line.empty() && line[0] == '%') continue;
        const char* p = line.data();
        const char* e = p + line.size();
        if (!(read_ll(p, e, rows) && read_ll(p, e, cols) && read_ll(p, e, nnz))) parse_fail(path, L.line_no, "size line");
        break;
      }
      if (rows != cols) parse_fail(path, L.line_no, "factor must be square");
      n = static_cast<std::int32_t>(rows);
      struct Rec {
        std::int32_t i, j;
        double v;
      };
      auto rec = [&](const char* p, const char* e, Rec& r) -> const char* {
        long long i = 0, j = 0;
        if (!(read_ll(p, e, i) && read_ll(p, e, j) && read_double(p, e, r.v))) return "malformed entry";
        if (i <= j || i > rows || j < 1) return "entry not strictly lower triangular";
        r.i = static_cast<std::int32_t>(i - 1);
        r.j = static_cast<std::int32_t>(j - 1);
        return nullptr;
      };
      const std::vector<Rec> recs = parse_records<Rec>(path, std::string_view(text).substr(L.pos), L.line_no,
                                                       std::max<long long>(nnz, 0), false, rec,
                                                       "unexpected end of file");
      // bucket by column in file order, then sort each column's (row, value)
      col_ptr.assign(static_cast<std::size_t>(std::max(n, 0)) + 1, 0);
      for (const Rec& r : recs) ++col_ptr[static_cast<std::size_t>(r.j) + 1];
      for (std::int32_t k = 0; k < n; ++k) col_ptr[k + 1] += col_ptr[k];
      std::vector<std::pair<std::int32_t, double>> ent(recs.size());
      {
        std::vector<std::int64_t> cur(col_ptr.begin(), col_ptr.end() - 1);
        for (const Rec& r : recs) ent[static_cast<std::size_t>(cur[r.j]++)] = {r.i, r.v};
      }
      split_run(n, host_threads(), [&](int, std::int64_t lo, std::int64_t hi) {
        for (std::int64_t k = lo; k < hi; ++k) std::sort(ent.begin() + col_ptr[k], ent.begin() + col_ptr[k + 1]);
      });
      rows_out.resize(ent.size());
      vals_out.resize(ent.size());
      for (std::size_t q = 0; q < ent.size(); ++q) {
        rows_out[q] = ent[q].first;
        vals_out[q] = ent[q].second;
      }
    }
    std::vector<double> diag;
    {
      const std::string path = stem + ".D.mtx";
      const std::string text = slurp(path);
      Lines L{text};
      std::string_view line;
      if (!L.next(line)) parse_fail(path, L.line_no, "empty file");
      if (line.rfind("%%MatrixMarket matrix array real", 0) != 0)
        throw Failure{unsupported_field, path + ": expected array real"};
      long long rows = 0, cols = 0;
      while (L.next(line)) {
        if (!line.empty() && line[0] == '%') continue;
        const char* p = line.data();
        const char* e = p + line.size();
        if (!(read_ll(p, e, rows) && read_ll(p, e, cols))) parse_fail(path, L.line_no, "size line");
        break;
      }
      if (rows != n || cols != 1) parse_fail(path, L.line_no, "diagonal length mismatch");
      auto rec = [&](const char* p, const char* e, double& v) -> const char* {
        return read_double(p, e, v) ? nullptr : "malformed value";
      };
      diag = parse_records<double>(path, std::string_view(text).substr(L.pos), L.line_no, rows, false, rec,
                                   "unexpected end of file");
    }
    std::vector<std::int32_t> perm;
    if (perm_path && perm_path[0]) {
      perm = read_positions(perm_path, n);
    } else {
      perm.resize(static_cast<std::size_t>(std::max(n, 0)));
      for (std::int32_t v = 0; v < n; ++v) perm[static_cast<std::size_t>(v)] = v;
    }
    out->n = n;
    out->nnz = col_ptr.empty() ? 0 : col_ptr.back();
    out->col_ptr = dup(col_ptr);
    out->rows = dup(rows_out);
    out->values = dup(vals_out);
    out->diag = dup(diag);
    out->perm = dup(perm);
  });
}

int parac_write_vector(const char* path, int64_t n, const double* values) {
  return guarded([&] {
    File f(path);
    Out h;
    h.str("%%MatrixMarket matrix array real general\n");
    h.i(n);
    h.str(" 1\n");
    f.put(h.s);
    write_parallel(f, n, nullptr, [&](Out& o, std::int64_t k) {
      o.d(values[k]);
      o.c('\n');
    });
  });
}

int parac_read_vector(const char* path_c, double** values, int64_t* n_out) {
  return guarded([&] {
    const std::string path(path_c ? path_c : "");
    const std::string text = slurp(path);
    Lines L{text};
    std::string_view line;
    if (!L.next(line)) parse_fail(path, L.line_no, "empty file");
    if (line.rfind("%%MatrixMarket matrix array real", 0) != 0)
      throw Failure{unsupported_field, path + ": expected array real"};
    long long rows = 0, cols = 0;
    while (L.next(line)) {
      if (!line.empty() && line[0] == '%') continue;
      const char* p = line.data();
      const char* e = p + line.size();
      if (!(read_ll(p, e, rows) && read_ll(p, e, cols))) parse_fail(path, L.line_no, "size line");
      break;
    }
    if (cols != 1) parse_fail(path, L.line_no, "expected a single column");
    auto rec = [&](const char* p, const char* e, double& v) -> const char* {
      return read_double(p, e, v) ? nullptr : "malformed value";
    };
    const std::vector<double> v = parse_records<double>(path, std::string_view(text).substr(L.pos), L.line_no,
                                                        std::max<long long>(rows, 0), false, rec,
                                                        "unexpected end of file");
    *values = dup(v);
    *n_out = static_cast<int64_t>(v.size());
  });
}

void parac_free_array(void* p) { std::free(p); }

int parac_write_permutation(const char* path, int32_t n, const int32_t* perm) {
  return guarded([&] {
    File f(path, "cannot write permutation file ");
    write_parallel(f, n, nullptr, [&](Out& o, std::int64_t v) {
      o.i(perm[v]);
      o.c('\n');
    });
  });
}

int parac_read_permutation(const char* path, int32_t n, int32_t* perm) {
  return guarded([&] {
    const std::vector<std::int32_t> p = read_positions(path ? path : "", n);
    if (n > 0) std::memcpy(perm, p.data(), sizeof(std::int32_t) * static_cast<std::size_t>(n));
  });
}

}  // extern "C"
