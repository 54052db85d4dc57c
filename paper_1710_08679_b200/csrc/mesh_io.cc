// mesh_io.cc — the on-disk formats either side of the solve.
//
//  * TSMESH 1 text meshes (mesh_io.hpp:13-96) and the Dirichlet sidecar
//    (mesh_io.hpp:38-42, 98-115): byte-identical output to write_mesh /
//    write_dirichlet, and read_mesh's parse + validate_mesh (mesh.hpp:75-113)
//    with the same ParseError / ValidationError positions and messages.
//  * TSVEC 1 solution vectors (solution_io.hpp:12-84), from/to host or device
//    memory; the device path streams through two pinned staging buffers so
//    the PCIe copy of one chunk overlaps the file I/O of the other.
//  * TSBMESH 1: this library's binary mesh (raw little-endian arrays behind a
//    text header) — a 135M-node TSMESH is tens of GB of text; the binary form
//    reads at file-system speed and is validated the same way.
//
// The reference does all of this in one host thread through iostreams. Here
// text is parsed and formatted in parallel (OpenMP) over fixed-size blocks of
// lines: formatting uses std::to_chars, which is specified to match printf's
// "%.17g" exactly (C++17 [charconv]); parsing replicates what
// `std::istringstream >> double / int` accepts (libstdc++ num_get: the
// longest [sign]digits[.digits][e[sign]digits] prefix, strtod, overflow to
// ±inf = failure), so both readers accept and reject the same lines.
#include <cuda_runtime.h>
#include <omp.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "mesh_io.h"

namespace tsg {

namespace {

[[noreturn]] void parse_error(const std::string& path, long line, const std::string& msg) {
  fail(TS_ERR_PARSE, path + ":" + std::to_string(line) + ": " + msg);
}

// atomic_write (io_util.hpp:21-49): write `<target>.tmp<pid>.<n>` next to the
// target, then rename over it; the temporary is removed on any failure.
class AtomicFile {
 public:
  explicit AtomicFile(const std::string& path) : target_(path) {
    static std::atomic<uint64_t> counter{0};
    namespace fs = std::filesystem;
    const fs::path t(path);
    tmp_ = (t.parent_path() / (t.filename().string() + ".tmp" + std::to_string(::getpid()) + "." +
                               std::to_string(counter.fetch_add(1))))
               .string();
    f_ = std::fopen(tmp_.c_str(), "wb");
    if (!f_) validation("cannot open for writing: " + tmp_);
  }
  AtomicFile(const AtomicFile&) = delete;
  AtomicFile& operator=(const AtomicFile&) = delete;
  void write(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f_) != n) validation("write failed: " + tmp_);
  }
  void write(const std::string& s) { write(s.data(), s.size()); }
  void commit() {
    const bool ok = std::fflush(f_) == 0;
    const bool closed = std::fclose(f_) == 0;
    f_ = nullptr;
    if (!ok || !closed) {
      std::remove(tmp_.c_str());
      validation("write failed: " + tmp_);
    }
    std::error_code ec;
    std::filesystem::rename(tmp_, target_, ec);
    if (ec) {
      std::filesystem::remove(tmp_, ec);
      validation("cannot rename " + tmp_ + " to " + target_);
    }
    done_ = true;
  }
  ~AtomicFile() {
    if (f_) std::fclose(f_);
    if (!done_) std::remove(tmp_.c_str());
  }

 private:
  std::string target_, tmp_;
  FILE* f_ = nullptr;
  bool done_ = false;
};

// ---------------------------------------------------------------- scanning
// A cursor over one line (no '\n' inside). The extractors mirror
// `istream >> x` on an istringstream of the line.
struct Cur {
  const char* p;
  const char* e;
};

inline void skip_ws(Cur& c) {
  while (c.p < c.e && std::isspace(static_cast<unsigned char>(*c.p))) ++c.p;
}

// operator>>(std::string&): the next run of non-space characters
bool get_word(Cur& c, std::string& w) {
  skip_ws(c);
  const char* b = c.p;
  while (c.p < c.e && !std::isspace(static_cast<unsigned char>(*c.p))) ++c.p;
  if (c.p == b) return false;
  w.assign(b, c.p);
  return true;
}

// operator>>(long&): [+-]digits, decimal. As in C++11 num_get, a failed
// extraction still stores: 0 when no digits were read, the saturated value
// on overflow (the TSVEC header relies on this: an unreadable "nodes" is 0).
bool get_i64(Cur& c, int64_t& v) {
  skip_ws(c);
  const char* q = c.p;
  bool neg = false;
  if (q < c.e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  const char* d0 = q;
  unsigned __int128 acc = 0;
  const unsigned __int128 lim = (unsigned __int128)INT64_MAX + 1;
  while (q < c.e && *q >= '0' && *q <= '9') {
    acc = acc * 10 + unsigned(*q - '0');
    if (acc > lim) acc = lim + 1;
    ++q;
  }
  c.p = q;
  if (q == d0) {
    v = 0;
    return false;
  }
  if (acc > (neg ? lim : lim - 1)) {
    v = neg ? INT64_MIN : INT64_MAX;
    return false;
  }
  v = neg ? static_cast<int64_t>(-static_cast<__int128>(acc)) : static_cast<int64_t>(acc);
  return true;
}

// operator>>(int&): the long extraction, then an int range check (saturating)
bool get_i32(Cur& c, int32_t& v) {
  int64_t x;
  const bool ok = get_i64(c, x);
  v = static_cast<int32_t>(std::clamp<int64_t>(x, INT32_MIN, INT32_MAX));
  return ok && x >= INT32_MIN && x <= INT32_MAX;
}

// operator>>(double&): num_get collects [+-]digits[.digits][(e|E)[+-]digits]
// (the exponent only after a mantissa digit), strtod must consume all of it,
// and an overflow to ±inf is a failure.
bool get_f64(Cur& c, double& v) {
  skip_ws(c);
  char buf[128];
  int n = 0;
  const char* q = c.p;
  auto put = [&](char ch) {
    if (n < 127) buf[n++] = ch;
  };
  if (q < c.e && (*q == '+' || *q == '-')) put(*q++);
  bool mant = false;
  while (q < c.e && *q >= '0' && *q <= '9') put(*q++), mant = true;
  if (q < c.e && *q == '.') {
    put(*q++);
    while (q < c.e && *q >= '0' && *q <= '9') put(*q++), mant = true;
  }
  if (mant && q < c.e && (*q == 'e' || *q == 'E')) {
    put(*q++);
    if (q < c.e && (*q == '+' || *q == '-')) put(*q++);
    while (q < c.e && *q >= '0' && *q <= '9') put(*q++);
  }
  c.p = q;
  if (n == 0 || n >= 127) return false;
  buf[n] = '\0';
  char* end = nullptr;
  const double x = std::strtod(buf, &end);
  if (end != buf + n || std::isinf(x)) return false;
  v = x;
  return true;
}

// ------------------------------------------------------------ line reader
// Streams a file in blocks of whole lines (std::getline semantics: the last
// line may lack its '\n'; a final '\n' does not start another line).
class LineBlocks {
 public:
  LineBlocks(const std::string& path, const char* what) : path_(path) {
    f_ = std::fopen(path.c_str(), "rb");
    if (!f_) validation(std::string("cannot open ") + what + " file: " + path);
  }
  ~LineBlocks() {
    if (f_) std::fclose(f_);
  }
  // next block: fills `starts`/`ends` with its complete lines; false at EOF
  bool next(std::vector<const char*>& starts, std::vector<const char*>& ends) {
    starts.clear();
    ends.clear();
    if (eof_ && keep_ == 0) return false;
    // move the carried partial line to the front, then fill the rest
    if (keep_ && keep_from_) std::memmove(buf_.data(), buf_.data() + keep_from_, keep_);
    size_t have = keep_;
    for (;;) {
      if (buf_.size() < have + kBlock) buf_.resize(have + kBlock);
      if (!eof_) {
        const size_t got = std::fread(buf_.data() + have, 1, kBlock, f_);
        have += got;
        if (got < kBlock) eof_ = true;
      }
      const char* b = buf_.data();
      const void* last = have ? memrchr(b, '\n', have) : nullptr;
      if (last || eof_) {
        const size_t cut = last ? static_cast<const char*>(last) - b + 1 : 0;
        size_t stop = cut;
        if (eof_ && have > cut) stop = have;  // unterminated final line
        const char* p = b;
        const char* endp = b + stop;
        while (p < endp) {
          const char* nl = static_cast<const char*>(std::memchr(p, '\n', endp - p));
          const char* le = nl ? nl : endp;
          starts.push_back(p);
          ends.push_back(le);
          p = nl ? nl + 1 : endp;
        }
        keep_from_ = stop;
        keep_ = have - stop;
        if (eof_) keep_ = 0;
        return !starts.empty() || !eof_;
      }
      // no newline yet in a non-final buffer: one long line, keep reading
    }
  }

 private:
  static constexpr size_t kBlock = size_t(64) << 20;
  std::string path_;
  FILE* f_ = nullptr;
  std::vector<char> buf_;
  size_t keep_ = 0, keep_from_ = 0;
  bool eof_ = false;
};

// first failing item of a parallel sweep (smallest index wins)
struct FirstFail {
  std::atomic<int64_t> at{INT64_MAX};
  void note(int64_t i) {
    int64_t cur = at.load(std::memory_order_relaxed);
    while (i < cur && !at.compare_exchange_weak(cur, i, std::memory_order_relaxed)) {
    }
  }
  bool any() const { return at.load() != INT64_MAX; }
};

double tet_volume(const double* a, const double* b, const double* c, const double* d) {
  // tet_volume (mesh.hpp:13-20): dot(b - a, cross(c - a, d - a)) / 6
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double cr[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2], v[0] * w[1] - v[1] * w[0]};
  return (u[0] * cr[0] + u[1] * cr[1] + u[2] * cr[2]) / 6.0;
}

// ------------------------------------------------------------ formatting
inline char* put_g17(char* o, double x) {
  // == snprintf("%.17g") (C++17 to_chars with chars_format::general, precision 17)
  return std::to_chars(o, o + 40, x, std::chars_format::general, 17).ptr;
}
inline char* put_int(char* o, int64_t x) { return std::to_chars(o, o + 24, x).ptr; }

// Format `count` records in parallel into per-thread strings (record order
// preserved), then append them to the file in order. `fmt(i, out)` writes
// record i at `out` and returns the end; `max_len` bounds one record.
template <typename F>
void write_records(AtomicFile& out, int64_t count, size_t max_len, F fmt) {
  constexpr int64_t kRound = int64_t(1) << 20;  // records per formatting round
  const int nt = std::max(1, omp_get_max_threads());
  std::vector<std::string> parts(nt);
  for (int64_t r0 = 0; r0 < count; r0 += kRound) {
    const int64_t r1 = std::min(count, r0 + kRound);
    for (auto& s : parts) s.clear();
#pragma omp parallel num_threads(nt)
    {
      const int t = omp_get_thread_num(), T = omp_get_num_threads();
      const int64_t a = r0 + (r1 - r0) * t / T, b = r0 + (r1 - r0) * (t + 1) / T;
      std::string& s = parts[t];
      s.resize(static_cast<size_t>(b - a) * max_len);
      char* o = s.data();
      for (int64_t i = a; i < b; ++i) o = fmt(i, o);
      s.resize(o - s.data());
    }
    for (auto& s : parts) out.write(s);
  }
}

}  // namespace

// validate_mesh (mesh.hpp:75-113): the first offending element (lowest id,
// checks in the reference's order within it) names the error.
void validate_mesh(const Mesh& m) {
  static constexpr int kEdge[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  const int64_t n = m.n_nodes();
  if (m.vertex_count < 0 || m.vertex_count > n) validation("mesh: vertex_count out of range");
  if (m.material_id.size() * 10 != m.tets10.size()) validation("mesh: inconsistent per-element array sizes");
  double scale = 0.0;
  const int64_t nc = static_cast<int64_t>(m.coords.size());
#pragma omp parallel for reduction(max : scale) schedule(static)
  for (int64_t i = 0; i < nc; ++i) scale = std::max(scale, std::abs(m.coords[i]));
  const double tol = 1e-12 * std::max(scale, 1.0);
  const int64_t E = m.n_elems();
  const int32_t* T = m.tets10.data();
  const double* X = m.coords.data();
  FirstFail first;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const int32_t* t = T + 10 * e;
    bool bad = false;
    for (int k = 0; k < 10; ++k) bad |= t[k] < 0 || t[k] >= n;
    if (!bad) {
      bad = tet_volume(X + 3 * size_t(t[0]), X + 3 * size_t(t[1]), X + 3 * size_t(t[2]), X + 3 * size_t(t[3])) <= 0.0;
      for (int k = 0; k < 6 && !bad; ++k) {
        const double* a = X + 3 * size_t(t[kEdge[k][0]]);
        const double* b = X + 3 * size_t(t[kEdge[k][1]]);
        const double* mid = X + 3 * size_t(t[4 + k]);
        const double d0 = mid[0] - 0.5 * (a[0] + b[0]), d1 = mid[1] - 0.5 * (a[1] + b[1]),
                     d2 = mid[2] - 0.5 * (a[2] + b[2]);
        bad = std::sqrt(d0 * d0 + d1 * d1 + d2 * d2) > tol;
      }
    }
    if (bad) first.note(e);
  }
  if (first.any()) {  // re-check the first failing element serially for its message
    const int64_t e = first.at.load();
    const int32_t* t = T + 10 * e;
    const std::string el = "mesh: element " + std::to_string(e);
    for (int k = 0; k < 10; ++k)
      if (t[k] < 0 || t[k] >= n) validation(el + " references node " + std::to_string(t[k]) + " out of range");
    if (tet_volume(X + 3 * size_t(t[0]), X + 3 * size_t(t[1]), X + 3 * size_t(t[2]), X + 3 * size_t(t[3])) <= 0.0)
      validation(el + " has non-positive volume");
    for (int k = 0; k < 6; ++k) {
      const double* a = X + 3 * size_t(t[kEdge[k][0]]);
      const double* b = X + 3 * size_t(t[kEdge[k][1]]);
      const double* mid = X + 3 * size_t(t[4 + k]);
      const double d0 = mid[0] - 0.5 * (a[0] + b[0]), d1 = mid[1] - 0.5 * (a[1] + b[1]),
                   d2 = mid[2] - 0.5 * (a[2] + b[2]);
      if (std::sqrt(d0 * d0 + d1 * d1 + d2 * d2) > tol)
        validation(el + " edge node " + std::to_string(t[4 + k]) + " is not at its edge midpoint");
    }
  }
  for (size_t i = 0; i < m.bc_node.size(); ++i)
    if (m.bc_node[i] < 0 || m.bc_node[i] >= n || m.bc_axis[i] < 0 || m.bc_axis[i] > 2)
      validation("mesh: dirichlet entry out of range");
}

// ------------------------------------------------------------ TSMESH text
void write_tsmesh(const Mesh& m, const std::string& path) {
  AtomicFile out(path);
  out.write("TSMESH 1\nnodes " + std::to_string(m.n_nodes()) + " vertex_nodes " + std::to_string(m.vertex_count) +
            " tets " + std::to_string(m.n_elems()) + "\n");
  const double* X = m.coords.data();
  write_records(out, m.n_nodes(), 3 * 26 + 1, [X](int64_t i, char* o) {
    o = put_g17(o, X[3 * i]);
    *o++ = ' ';
    o = put_g17(o, X[3 * i + 1]);
    *o++ = ' ';
    o = put_g17(o, X[3 * i + 2]);
    *o++ = '\n';
    return o;
  });
  const int32_t* T = m.tets10.data();
  const int32_t* M = m.material_id.data();
  write_records(out, m.n_elems(), 11 * 12 + 1, [T, M](int64_t e, char* o) {
    for (int k = 0; k < 10; ++k) {
      o = put_int(o, T[10 * e + k]);
      *o++ = ' ';
    }
    o = put_int(o, M[e]);
    *o++ = '\n';
    return o;
  });
  out.commit();
}

Mesh read_tsmesh(const std::string& path) {
  LineBlocks in(path, "mesh");
  std::vector<const char*> ls, le;
  Mesh m;
  int64_t n_nodes = -1, n_verts = -1, n_tets = -1;
  int64_t lineno = 0;  // lines consumed so far
  int64_t need = 2;    // header lines, then grown to 2 + N + T
  while (lineno < need && in.next(ls, le)) {
    size_t i = 0;
    // header lines (sequential, at most the first two lines of the file)
    while (i < ls.size() && lineno < 2) {
      Cur c{ls[i], le[i]};
      ++lineno;
      if (lineno == 1) {
        std::string magic;
        int32_t version = 0;
        get_word(c, magic) && get_i32(c, version);
        if (magic != "TSMESH" || version != 1) parse_error(path, lineno, "expected header 'TSMESH 1'");
      } else {
        std::string k1, k2, k3;
        const bool ok = get_word(c, k1) && get_i64(c, n_nodes) && get_word(c, k2) && get_i64(c, n_verts) &&
                        get_word(c, k3) && get_i64(c, n_tets);
        if (k1 != "nodes" || k2 != "vertex_nodes" || k3 != "tets" || !ok || n_nodes < 0 || n_verts < 0 ||
            n_tets < 0)
          parse_error(path, lineno, "expected 'nodes N vertex_nodes V tets T'");
        m.vertex_count = static_cast<int32_t>(n_verts);
        m.coords.resize(3 * static_cast<size_t>(n_nodes));
        m.tets10.resize(10 * static_cast<size_t>(n_tets));
        m.material_id.resize(static_cast<size_t>(n_tets));
        need = 2 + n_nodes + n_tets;
      }
      ++i;
    }
    // body lines of this block in parallel: line g (0-based) is node g-2 or element g-2-N
    const int64_t base = lineno - static_cast<int64_t>(i);  // global index of ls[0]
    const int64_t count = std::min<int64_t>(static_cast<int64_t>(ls.size()), need - base);
    FirstFail bad;
    double* X = m.coords.data();
    int32_t* T = m.tets10.data();
    int32_t* M = m.material_id.data();
#pragma omp parallel for schedule(static)
    for (int64_t j = static_cast<int64_t>(i); j < count; ++j) {
      const int64_t g = base + j;
      Cur c{ls[j], le[j]};
      bool ok;
      if (g < 2 + n_nodes) {
        double* x = X + 3 * (g - 2);
        ok = get_f64(c, x[0]) && get_f64(c, x[1]) && get_f64(c, x[2]);
      } else {
        const int64_t e = g - 2 - n_nodes;
        ok = true;
        for (int k = 0; k < 10 && ok; ++k) ok = get_i32(c, T[10 * e + k]);
        ok = ok && get_i32(c, M[e]);
      }
      if (!ok) bad.note(g);
    }
    if (bad.any()) {
      const int64_t g = bad.at.load();
      if (g < 2 + n_nodes) parse_error(path, g + 1, "expected 3 node coordinates");
      parse_error(path, g + 1,
                  "expected 10 node ids and a material id for element " + std::to_string(g - 2 - n_nodes));
    }
    lineno = std::max<int64_t>(lineno, base + count);
  }
  if (lineno < need) parse_error(path, lineno + 1, "unexpected end of file");
  validate_mesh(m);
  return m;
}

void write_dirichlet(const Mesh& m, const std::string& path) {
  AtomicFile out(path);
  const int32_t* N = m.bc_node.data();
  const int8_t* A = m.bc_axis.data();
  write_records(out, static_cast<int64_t>(m.bc_node.size()), 16, [N, A](int64_t i, char* o) {
    o = put_int(o, N[i]);
    *o++ = ' ';
    o = put_int(o, A[i]);
    *o++ = '\n';
    return o;
  });
  out.commit();
}

void read_dirichlet(Mesh& m, const std::string& path) {
  LineBlocks in(path, "dirichlet");
  std::vector<const char*> ls, le;
  std::vector<int32_t> node;
  std::vector<int8_t> axis;
  const int64_t n = m.n_nodes();
  int64_t lineno = 0;
  while (in.next(ls, le)) {
    const int64_t L = static_cast<int64_t>(ls.size());
    std::vector<int32_t> bn(L);
    std::vector<int8_t> ba(L), keep(L);
    FirstFail bad;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < L; ++j) {
      if (ls[j] == le[j]) continue;  // empty lines are skipped
      Cur c{ls[j], le[j]};
      int64_t nd = -1;
      int32_t ax = -1;
      const bool ok = get_i64(c, nd) && get_i32(c, ax);
      if (!ok || nd < 0 || nd >= n || ax < 0 || ax > 2) {
        bad.note(j);
        continue;
      }
      bn[j] = static_cast<int32_t>(nd);
      ba[j] = static_cast<int8_t>(ax);
      keep[j] = 1;
    }
    if (bad.any()) parse_error(path, lineno + bad.at.load() + 1, "expected 'node_id axis' with axis in 0..2");
    for (int64_t j = 0; j < L; ++j)
      if (keep[j]) node.push_back(bn[j]), axis.push_back(ba[j]);
    lineno += L;
  }
  m.bc_node.swap(node);
  m.bc_axis.swap(axis);
}

// ------------------------------------------------------------ TSBMESH binary
// "TSBMESH 1\nnodes N vertex_nodes V tets T dirichlet D\nendian little\nDATA\n"
// then coords f64[N][3], tets10 i32[T][10], material i32[T], bc_node i32[D], bc_axis i8[D].
void write_tsbmesh(const Mesh& m, const std::string& path) {
  AtomicFile out(path);
  out.write("TSBMESH 1\nnodes " + std::to_string(m.n_nodes()) + " vertex_nodes " + std::to_string(m.vertex_count) +
            " tets " + std::to_string(m.n_elems()) + " dirichlet " + std::to_string(m.bc_node.size()) +
            "\nendian little\nDATA\n");
  out.write(m.coords.data(), m.coords.size() * sizeof(double));
  out.write(m.tets10.data(), m.tets10.size() * sizeof(int32_t));
  out.write(m.material_id.data(), m.material_id.size() * sizeof(int32_t));
  out.write(m.bc_node.data(), m.bc_node.size() * sizeof(int32_t));
  out.write(m.bc_axis.data(), m.bc_axis.size());
  out.commit();
}

namespace {
// read one '\n'-terminated header line (<= 4 KB) from a binary file
bool header_line(FILE* f, std::string& line) {
  line.clear();
  for (int c; (c = std::fgetc(f)) != EOF;) {
    if (c == '\n') return true;
    if (line.size() > 4096) return false;
    line.push_back(static_cast<char>(c));
  }
  return !line.empty();
}

// fread in large pieces, each thread reading its own slice (pread) so big
// arrays load at storage bandwidth
bool read_exact(FILE* f, void* dst, size_t bytes) {
  if (!bytes) return true;
  const int fd = fileno(f);
  const off_t at = ftello(f);
  constexpr size_t kSlice = size_t(64) << 20;
  const int64_t n = static_cast<int64_t>((bytes + kSlice - 1) / kSlice);
  std::atomic<bool> ok{true};
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < n; ++s) {
    const size_t off = static_cast<size_t>(s) * kSlice, len = std::min(kSlice, bytes - off);
    size_t done = 0;
    while (done < len) {
      const ssize_t r = ::pread(fd, static_cast<char*>(dst) + off + done, len - done, at + off_t(off + done));
      if (r <= 0) {
        ok = false;
        break;
      }
      done += static_cast<size_t>(r);
    }
  }
  std::fseek(f, at + off_t(bytes), SEEK_SET);
  return ok;
}
}  // namespace

Mesh read_tsbmesh(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) validation("cannot open mesh file: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  std::string line;
  long lineno = 0;
  auto expect = [&](const char* what) {
    if (!header_line(f, line)) parse_error(path, lineno + 1, "unexpected end of file");
    ++lineno;
    Cur c{line.data(), line.data() + line.size()};
    std::string key;
    get_word(c, key);
    if (key != what) parse_error(path, lineno, std::string("expected '") + what + "' header line");
    return c;
  };
  {
    Cur c = expect("TSBMESH");
    int32_t v = 0;
    if (!get_i32(c, v) || v != 1) parse_error(path, lineno, "unsupported version");
  }
  int64_t nn = -1, nv = -1, ne = -1, nd = -1;
  {
    Cur c = expect("nodes");
    std::string k2, k3, k4;
    const bool ok = get_i64(c, nn) && get_word(c, k2) && get_i64(c, nv) && get_word(c, k3) && get_i64(c, ne) &&
                    get_word(c, k4) && get_i64(c, nd);
    if (!ok || k2 != "vertex_nodes" || k3 != "tets" || k4 != "dirichlet" || nn < 0 || nv < 0 || ne < 0 || nd < 0 ||
        nn >= (int64_t(1) << 31) || ne >= (int64_t(1) << 31))
      parse_error(path, lineno, "expected 'nodes N vertex_nodes V tets T dirichlet D'");
  }
  {
    Cur c = expect("endian");
    std::string e;
    get_word(c, e);
    if (e != "little") parse_error(path, lineno, "expected little endian");
  }
  expect("DATA");
  Mesh m;
  m.vertex_count = static_cast<int32_t>(nv);
  m.coords.resize(3 * size_t(nn));
  m.tets10.resize(10 * size_t(ne));
  m.material_id.resize(size_t(ne));
  m.bc_node.resize(size_t(nd));
  m.bc_axis.resize(size_t(nd));
  const bool ok = read_exact(f, m.coords.data(), m.coords.size() * sizeof(double)) &&
                  read_exact(f, m.tets10.data(), m.tets10.size() * sizeof(int32_t)) &&
                  read_exact(f, m.material_id.data(), m.material_id.size() * sizeof(int32_t)) &&
                  read_exact(f, m.bc_node.data(), m.bc_node.size() * sizeof(int32_t)) &&
                  read_exact(f, m.bc_axis.data(), m.bc_axis.size());
  if (!ok) parse_error(path, lineno + 1, "truncated binary payload");
  validate_mesh(m);
  return m;
}

// ------------------------------------------------------------ TSVEC
namespace {
std::string tsvec_header(int64_t nodes, int64_t batch) {
  return "TSVEC 1\nnodes " + std::to_string(nodes) + "\naxes 3\nbatch " + std::to_string(batch) +
         "\nprecision float64\nendian little\norder node_axis_batch\nDATA\n";
}

// pinned double-buffered staging between a device array and a file
struct Staging {
  static constexpr size_t kChunk = size_t(64) << 20;
  void* h[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  Staging() {
    require_device();
    for (int i = 0; i < 2; ++i) {
      TS_CUDA(cudaMallocHost(&h[i], kChunk));
      TS_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    TS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~Staging() {
    if (s) cudaStreamSynchronize(s), cudaStreamDestroy(s);
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (h[i]) cudaFreeHost(h[i]);
    }
  }
};
}  // namespace

void write_tsvec(const std::string& path, const double* u, int64_t nodes, int64_t batch, bool on_device) {
  if (nodes < 0 || batch < 1) validation("solution: bad dimensions");
  AtomicFile out(path);
  out.write(tsvec_header(nodes, batch));
  const size_t bytes = 3 * size_t(nodes) * size_t(batch) * sizeof(double);
  if (!on_device) {
    out.write(u, bytes);
  } else if (bytes) {
    // D2H of chunk k+1 overlaps the file write of chunk k
    Staging st;
    const size_t n = (bytes + Staging::kChunk - 1) / Staging::kChunk;
    auto copy = [&](size_t k) {
      const size_t off = k * Staging::kChunk, len = std::min(Staging::kChunk, bytes - off);
      TS_CUDA(cudaMemcpyAsync(st.h[k & 1], reinterpret_cast<const char*>(u) + off, len, cudaMemcpyDeviceToHost, st.s));
      TS_CUDA(cudaEventRecord(st.ev[k & 1], st.s));
    };
    copy(0);
    for (size_t k = 0; k < n; ++k) {
      if (k + 1 < n) copy(k + 1);  // its buffer was written out (synchronously) at iteration k-1
      TS_CUDA(cudaEventSynchronize(st.ev[k & 1]));
      const size_t off = k * Staging::kChunk, len = std::min(Staging::kChunk, bytes - off);
      out.write(st.h[k & 1], len);
    }
  }
  out.commit();
}

void tsvec_info(const std::string& path, int64_t* nodes, int64_t* batch, int64_t* data_offset) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) validation("cannot open solution file: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  std::string line;
  long lineno = 0;
  auto expect = [&](const char* what) {
    if (!header_line(f, line)) parse_error(path, lineno + 1, "unexpected end of file");
    ++lineno;
    Cur c{line.data(), line.data() + line.size()};
    std::string key;
    get_word(c, key);
    if (key != what) parse_error(path, lineno, std::string("expected '") + what + "' header line");
    return c;
  };
  // solution_io.hpp:43-77, same checks in the same order
  {
    Cur c = expect("TSVEC");
    int32_t v = 0;
    get_i32(c, v);
    if (v != 1) parse_error(path, lineno, "unsupported version");
  }
  int64_t nn = -1, nb = -1;
  {
    Cur c = expect("nodes");
    get_i64(c, nn);
  }
  {
    Cur c = expect("axes");
    int32_t a = 0;
    get_i32(c, a);
    if (a != 3) parse_error(path, lineno, "expected 3 axes");
  }
  {
    Cur c = expect("batch");
    get_i64(c, nb);
  }
  {
    Cur c = expect("precision");
    std::string p;
    get_word(c, p);
    if (p != "float64") parse_error(path, lineno, "expected float64 precision");
  }
  {
    Cur c = expect("endian");
    std::string e;
    get_word(c, e);
    if (e != "little") parse_error(path, lineno, "expected little endian");
  }
  {
    Cur c = expect("order");
    std::string o;
    get_word(c, o);
    if (o != "node_axis_batch") parse_error(path, lineno, "unexpected layout order");
  }
  expect("DATA");
  if (nn < 0 || nb < 1) parse_error(path, lineno, "bad dimensions");
  *nodes = nn;
  *batch = nb;
  *data_offset = ftello(f);
}

void read_tsvec(const std::string& path, double* u, int64_t nodes, int64_t batch, bool on_device) {
  int64_t nn, nb, off;
  tsvec_info(path, &nn, &nb, &off);
  if (nn != nodes || nb != batch)
    validation("solution file " + path + " holds " + std::to_string(nn) + " nodes x " + std::to_string(nb) +
               " cases, caller expects " + std::to_string(nodes) + " x " + std::to_string(batch));
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) validation("cannot open solution file: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  std::fseek(f, off, SEEK_SET);
  const size_t bytes = 3 * size_t(nodes) * size_t(batch) * sizeof(double);
  if (!on_device) {
    if (!read_exact(f, u, bytes)) parse_error(path, 9, "truncated binary payload");
    return;
  }
  if (!bytes) return;
  // file read of chunk k+1 overlaps the H2D copy of chunk k
  Staging st;
  const size_t n = (bytes + Staging::kChunk - 1) / Staging::kChunk;
  for (size_t k = 0; k < n; ++k) {
    const size_t o = k * Staging::kChunk, len = std::min(Staging::kChunk, bytes - o);
    if (k >= 2) TS_CUDA(cudaEventSynchronize(st.ev[k & 1]));  // buffer free again
    if (std::fread(st.h[k & 1], 1, len, f) != len) {
      TS_CUDA(cudaStreamSynchronize(st.s));
      parse_error(path, 9, "truncated binary payload");
    }
    TS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(u) + o, st.h[k & 1], len, cudaMemcpyHostToDevice, st.s));
    TS_CUDA(cudaEventRecord(st.ev[k & 1], st.s));
  }
  TS_CUDA(cudaStreamSynchronize(st.s));
}

// ------------------------------------------------------------ Green's-sweep files
// TSFAULT 1 (fault.hpp:44-84, 414-419), observation lists (greens.hpp:20-44) and
// TSGREENS 1 banks (greens.hpp:147-222): same bytes on write, same accept /
// reject (ParseError line and message) on read.
namespace {
std::string g17(double x) {
  char b[40];
  return std::string(b, put_g17(b, x));
}
// whole-file line reader for the small Green's files (std::getline semantics)
struct Lines {
  std::vector<char> buf;
  std::vector<std::pair<const char*, const char*>> lines;
  Lines(const std::string& path, const char* what, bool binary_tail = false) {
    (void)binary_tail;
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) validation(std::string("cannot open ") + what + ": " + path);
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize(size_t(std::max(0L, n)));
    const size_t got = n > 0 ? std::fread(buf.data(), 1, size_t(n), f) : 0;
    std::fclose(f);
    buf.resize(got);
    const char* p = buf.data();
    const char* e = p + buf.size();
    while (p < e) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', e - p));
      lines.push_back({p, nl ? nl : e});
      p = nl ? nl + 1 : e;
    }
  }
};
}  // namespace

void write_fault_faces(const std::vector<std::array<int32_t, 3>>& faces, const std::string& path) {
  AtomicFile out(path);
  std::string s = "TSFAULT 1\nfaces " + std::to_string(faces.size()) + "\n";
  char b[48];
  for (const auto& f : faces) {
    char* o = put_int(b, f[0]);
    *o++ = ' ';
    o = put_int(o, f[1]);
    *o++ = ' ';
    o = put_int(o, f[2]);
    *o++ = '\n';
    s.append(b, o);
  }
  out.write(s);
  out.commit();
}

std::vector<std::array<int32_t, 3>> read_fault_faces(const std::string& path) {
  Lines L(path, "fault file");
  size_t li = 0;
  auto next = [&]() {
    if (li >= L.lines.size()) parse_error(path, long(li) + 1, "unexpected end of file");
    const auto [a, b] = L.lines[li++];
    return Cur{a, b};
  };
  {
    Cur c = next();
    std::string magic;
    int32_t ver = 0;
    get_word(c, magic) && get_i32(c, ver);
    if (magic != "TSFAULT" || ver != 1) parse_error(path, long(li), "expected 'TSFAULT 1'");
  }
  int64_t n = -1;
  {
    Cur c = next();
    std::string k;
    const bool ok = get_word(c, k) && get_i64(c, n);
    if (k != "faces" || !ok || n < 1) parse_error(path, long(li), "expected 'faces F'");
  }
  std::vector<std::array<int32_t, 3>> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Cur c = next();
    if (!(get_i32(c, out[i][0]) && get_i32(c, out[i][1]) && get_i32(c, out[i][2])))
      parse_error(path, long(li), "expected 3 vertex ids");
  }
  return out;
}

std::vector<Observation> read_observations(const std::string& path) {
  Lines L(path, "observations file");
  std::vector<Observation> out;
  for (size_t li = 0; li < L.lines.size(); ++li) {
    const char* a = L.lines[li].first;
    const char* b = L.lines[li].second;
    const char* hash = static_cast<const char*>(std::memchr(a, '#', b - a));
    Cur c{a, hash ? hash : b};
    Observation o;
    if (!get_f64(c, o.p[0])) continue;  // blank, comment or non-numeric lines are skipped
    std::string ax;
    if (!(get_f64(c, o.p[1]) && get_f64(c, o.p[2]) && get_word(c, ax)))
      parse_error(path, long(li) + 1, "expected 'x y z axis'");
    if (ax == "x" || ax == "0") o.axis = 0;
    else if (ax == "y" || ax == "1") o.axis = 1;
    else if (ax == "z" || ax == "2") o.axis = 2;
    else parse_error(path, long(li) + 1, "axis must be one of x, y, z or 0..2");
    out.push_back(o);
  }
  if (out.empty()) validation(path + ": no observation components");
  return out;
}

void write_greens_bank(const GreensBankData& g, const std::string& path) {
  AtomicFile out(path);
  std::string s = "TSGREENS 1\nrows " + std::to_string(g.rows) + " cols " + std::to_string(g.cols) + "\n";
  for (int32_t r = 0; r < g.rows; ++r)
    s += "obs " + g17(g.obs[r].p[0]) + ' ' + g17(g.obs[r].p[1]) + ' ' + g17(g.obs[r].p[2]) + ' ' +
         std::to_string(g.obs[r].axis) + "\n";
  for (int32_t c = 0; c < g.cols; ++c)
    s += "col " + g17(g.centers[3 * size_t(c)]) + ' ' + g17(g.centers[3 * size_t(c) + 1]) + ' ' +
         g17(g.centers[3 * size_t(c) + 2]) + ' ' + (g.dirs[c] == 0 ? "dip" : "strike") + ' ' + g17(g.radii[c]) + "\n";
  s += "DATA\n";
  out.write(s);
  out.write(g.values.data(), g.values.size() * sizeof(double));
  out.commit();
}

GreensBankData read_greens_bank(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) validation("cannot open greens bank: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  GreensBankData g;
  std::string line;
  long lineno = 0;
  auto next = [&]() {
    if (!header_line(f, line)) parse_error(path, lineno + 1, "unexpected end of file");
    ++lineno;
    return Cur{line.data(), line.data() + line.size()};
  };
  {
    Cur c = next();
    std::string magic;
    int32_t ver = 0;
    get_word(c, magic) && get_i32(c, ver);
    if (magic != "TSGREENS" || ver != 1) parse_error(path, lineno, "expected 'TSGREENS 1'");
  }
  {
    Cur c = next();
    std::string k1, k2;
    const bool ok = get_word(c, k1) && get_i32(c, g.rows) && get_word(c, k2) && get_i32(c, g.cols);
    if (k1 != "rows" || k2 != "cols" || !ok || g.rows < 1 || g.cols < 1)
      parse_error(path, lineno, "expected 'rows M cols N'");
  }
  for (int32_t r = 0; r < g.rows; ++r) {
    Cur c = next();
    std::string tag;
    Observation o;
    const bool ok = get_word(c, tag) && get_f64(c, o.p[0]) && get_f64(c, o.p[1]) && get_f64(c, o.p[2]) &&
                    get_i32(c, o.axis);
    if (tag != "obs" || !ok) parse_error(path, lineno, "expected 'obs x y z axis'");
    g.obs.push_back(o);
  }
  for (int32_t col = 0; col < g.cols; ++col) {
    Cur c = next();
    std::string tag, dir;
    double x[3], rad = 0.0;
    const bool ok = get_word(c, tag) && get_f64(c, x[0]) && get_f64(c, x[1]) && get_f64(c, x[2]) &&
                    get_word(c, dir) && get_f64(c, rad);
    if (tag != "col" || !ok || (dir != "dip" && dir != "strike"))
      parse_error(path, lineno, "expected 'col x y z dip|strike radius'");
    g.centers.insert(g.centers.end(), x, x + 3);
    g.dirs.push_back(dir == "dip" ? 0 : 1);
    g.radii.push_back(rad);
  }
  {
    Cur c = next();
    std::string tag;
    get_word(c, tag);
    if (tag != "DATA") parse_error(path, lineno, "expected 'DATA'");
  }
  g.values.resize(size_t(g.rows) * g.cols);
  const size_t bytes = g.values.size() * sizeof(double);
  if (std::fread(g.values.data(), 1, bytes, f) != bytes) parse_error(path, lineno + 1, "truncated binary matrix payload");
  return g;
}

}  // namespace tsg
