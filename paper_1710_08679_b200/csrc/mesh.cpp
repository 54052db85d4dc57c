#include <chrono>
#include <cstdio>
#include <cstdlib>
// mesh.cpp — host mesh container and the layered box generator.
//
// generate_box_mesh reproduces the reference numbering exactly
// (box_mesh.hpp:55-157): vertices lexicographic in (z, y, x), six Kuhn tets
// per cell from the six axis orderings, v2/v3 swapped for positive volume,
// then edge midpoints numbered in element discovery order with local edges
// (0,1),(1,2),(2,0),(0,3),(1,3),(2,3). The reference finds edges with a
// std::map; here every Kuhn edge joins two corners of one cell, so an edge is
// keyed by (lower vertex, 3-bit axis offset) in a dense table — O(1), no tree,
// same discovery order, same ids.
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstring>
#include <omp.h>

#include "ts_common.h"

namespace tsg {

namespace {
thread_local std::string g_last_error;

double tet_volume(const double* a, const double* b, const double* c, const double* d) {
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double cr[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2],
                        v[0] * w[1] - v[1] * w[0]};
  return (u[0] * cr[0] + u[1] * cr[1] + u[2] * cr[2]) / 6.0;
}
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }
const std::string& last_error() { return g_last_error; }

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n < 1)
    fail(TS_ERR_CUDA, std::string("no CUDA device available (libtsgpu has no CPU fallback): ") +
                          cudaGetErrorString(e));
}

std::vector<uint8_t> Mesh::dirichlet_mask() const {
  std::vector<uint8_t> mask(3 * static_cast<size_t>(n_nodes()), 0);
  for (size_t i = 0; i < bc_node.size(); ++i) mask[3 * size_t(bc_node[i]) + bc_axis[i]] = 1;
  return mask;
}

Mesh generate_box_mesh(const double ext[3], const int32_t div[3],
                       const std::vector<double>& interfaces, int fixed) {
  for (int a = 0; a < 3; ++a) {
    if (ext[a] <= 0.0)
      validation("box mesh spec: extents must be positive, got " + std::to_string(ext[a]) +
                 " on axis " + std::to_string(a));
    if (div[a] < 1)
      validation("box mesh spec: divisions must be >= 1, got " + std::to_string(div[a]) +
                 " on axis " + std::to_string(a));
  }
  double prev = 0.0;
  for (double z : interfaces) {
    if (z <= prev || z >= ext[2])
      validation("box mesh spec: layer interfaces must be strictly increasing and interior to (0, Lz)");
    prev = z;
  }
  const int64_t nx = div[0], ny = div[1], nz = div[2];
  const int64_t nv = (nx + 1) * (ny + 1) * (nz + 1);
  const int64_t ne = 6 * nx * ny * nz;
  if (nv > (int64_t(1) << 28) || ne > INT32_MAX / 2) validation("box mesh: too large for int32 ids");
  const double hx = ext[0] / nx, hy = ext[1] / ny, hz = ext[2] / nz;

  Mesh m;
  m.vertex_count = static_cast<int32_t>(nv);
  static constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                      {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static constexpr int edge_ends[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  const int n_layers = static_cast<int>(interfaces.size()) + 1;
  HostVec<double> vxyz(3 * static_cast<size_t>(nv));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < nv; ++v) {
    const int64_t i = v % (nx + 1), j = (v / (nx + 1)) % (ny + 1), k = v / ((nx + 1) * (ny + 1));
    vxyz[3 * v] = i * hx;
    vxyz[3 * v + 1] = j * hy;
    vxyz[3 * v + 2] = k * hz;
  }
  m.tets10.resize(10 * static_cast<size_t>(ne));
  m.material_id.resize(static_cast<size_t>(ne));
  auto vid = [&](int64_t i, int64_t j, int64_t k) { return i + (nx + 1) * (j + (ny + 1) * k); };
  // six Kuhn tets per cell, cells in (z, y, x) order: independent per cell
#pragma omp parallel for schedule(static)
  for (int64_t cell = 0; cell < nx * ny * nz; ++cell) {
    const int64_t i = cell % nx, j = (cell / nx) % ny, k = cell / (nx * ny);
    for (int pp = 0; pp < 6; ++pp) {
      const auto& p = perms[pp];
      int64_t corner[4][3] = {{i, j, k}, {}, {}, {}};
      for (int st = 0; st < 3; ++st) {
        for (int ax = 0; ax < 3; ++ax) corner[st + 1][ax] = corner[st][ax];
        corner[st + 1][p[st]] += 1;
      }
      int32_t v[4];
      for (int st = 0; st < 4; ++st) v[st] = static_cast<int32_t>(vid(corner[st][0], corner[st][1], corner[st][2]));
      const double* c = vxyz.data();
      if (tet_volume(c + 3 * size_t(v[0]), c + 3 * size_t(v[1]), c + 3 * size_t(v[2]), c + 3 * size_t(v[3])) < 0.0)
        std::swap(v[2], v[3]);
      const size_t e = 6 * static_cast<size_t>(cell) + pp;
      int32_t* t = m.tets10.data() + 10 * e;
      for (int st = 0; st < 4; ++st) t[st] = v[st];
      const double zc = (c[3 * size_t(v[0]) + 2] + c[3 * size_t(v[1]) + 2] + c[3 * size_t(v[2]) + 2] +
                         c[3 * size_t(v[3]) + 2]) / 4.0;
      int below = 0;
      for (double z : interfaces)
        if (zc > z) ++below;
      m.material_id[e] = n_layers - 1 - below;  // layer 0 on top (box_mesh.hpp:75-82)
    }
  }
  // Edge midpoints, numbered in discovery order (element order, local edges
  // (0,1),(1,2),(2,0),(0,3),(1,3),(2,3)). An edge is keyed by (lower vertex,
  // 3-bit axis offset) in a dense table; in parallel: each edge keeps its first
  // occurrence (atomic min over the occurrence index 6e + s), the first
  // occurrences are counted by an ordered prefix sum, and every occurrence then
  // reads its edge's id — the same ids as the sequential scan.
  const int64_t sx = nx + 1, sxy = (nx + 1) * (ny + 1);
  const int64_t occ = 6 * ne;
  // key of occurrence q = 6e + s: a Kuhn edge joins two corners of one cell, so the id
  // difference is one of 7 values (no divisions)
  HostVec<uint32_t> keys(static_cast<size_t>(occ));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t* t = m.tets10.data() + 10 * e;
    for (int s2 = 0; s2 < 6; ++s2) {
      const int32_t a = t[edge_ends[s2][0]], b = t[edge_ends[s2][1]];
      const int64_t lo = std::min(a, b), d = std::max(a, b) - lo;
      const uint32_t bits = d == 1 ? 1u : d == sx ? 2u : d == sxy ? 4u : d == 1 + sx ? 3u : d == 1 + sxy ? 5u
                          : d == sx + sxy ? 6u : 7u;
      keys[6 * e + s2] = static_cast<uint32_t>(lo * 8 + bits);
    }
  }
  HostVec<int64_t> first(static_cast<size_t>(nv) * 8);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nv * 8; ++k) first[k] = INT64_MAX;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < occ; ++q) {
    int64_t* slot = &first[keys[q]];
    int64_t cur = __atomic_load_n(slot, __ATOMIC_RELAXED);
    while (q < cur && !__atomic_compare_exchange_n(slot, &cur, q, true, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
  }
  // ordered count of first occurrences: per-thread block sums, then an exclusive scan
  const int nt = std::max(1, omp_get_max_threads());
  std::vector<int64_t> part(nt + 1, 0);
#pragma omp parallel num_threads(nt)
  {
    const int tid = omp_get_thread_num(), T = omp_get_num_threads();
    const int64_t lo = occ * tid / T, hi = occ * (tid + 1) / T;
    int64_t c = 0;
    for (int64_t q = lo; q < hi; ++q) c += first[keys[q]] == q;
    part[tid + 1] = c;
#pragma omp barrier
#pragma omp single
    for (int u = 0; u < T; ++u) part[u + 1] += part[u];
    // first occurrences get ids nv + rank; the id is stored back in the key's slot (as -(id + 1))
    int64_t id = nv + part[tid];
    for (int64_t q = lo; q < hi; ++q)
      if (first[keys[q]] == q) m.tets10[10 * (q / 6) + 4 + q % 6] = static_cast<int32_t>(id++);
  }
  const int64_t n_edges = part[nt];
  if (nv + n_edges > (int64_t(1) << 28)) validation("box mesh: too large for int32 ids");
  // every occurrence reads the id its edge's first occurrence received
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < occ; ++q) {
    const int64_t f0 = first[keys[q]];
    if (f0 != q) m.tets10[10 * (q / 6) + 4 + q % 6] = m.tets10[10 * (f0 / 6) + 4 + f0 % 6];
  }
  const int32_t nn = static_cast<int32_t>(nv + n_edges);
  m.coords.resize(3 * static_cast<size_t>(nn));
  std::copy(vxyz.begin(), vxyz.end(), m.coords.begin());
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < occ; ++q) {
    const int32_t* t = m.tets10.data() + 10 * (q / 6);
    const int s = static_cast<int>(q % 6);
    if (first[keys[q]] != q) continue;
    const int32_t a = t[edge_ends[s][0]], b = t[edge_ends[s][1]], id = t[4 + s];
    for (int cc = 0; cc < 3; ++cc)
      m.coords[3 * size_t(id) + cc] = 0.5 * (m.coords[3 * size_t(a) + cc] + m.coords[3 * size_t(b) + cc]);
  }
  // Dirichlet set by node coordinate (box_mesh.hpp:134-155), built per thread on contiguous node
  // ranges and concatenated in node order (the sequential list)
  if (fixed != 0) {
    const double tol = 1e-9 * std::max({ext[0], ext[1], ext[2]});
    const int T = std::max(1, omp_get_max_threads());
    std::vector<std::vector<int32_t>> bn(T);
    std::vector<std::vector<int8_t>> ba(T);
#pragma omp parallel num_threads(T)
    {
      const int tid = omp_get_thread_num(), TT = omp_get_num_threads();
      const int32_t lo = static_cast<int32_t>(int64_t(nn) * tid / TT);
      const int32_t hi = static_cast<int32_t>(int64_t(nn) * (tid + 1) / TT);
      auto& N = bn[tid];
      auto& A = ba[tid];
      for (int32_t n = lo; n < hi; ++n) {
        const double* c = m.coords.data() + 3 * size_t(n);
        const bool on_bottom = std::abs(c[2]) <= tol;
        const bool on_top = std::abs(c[2] - ext[2]) <= tol;
        const bool on_x = std::abs(c[0]) <= tol || std::abs(c[0] - ext[0]) <= tol;
        const bool on_y = std::abs(c[1]) <= tol || std::abs(c[1] - ext[1]) <= tol;
        auto push = [&](int8_t ax) {
          N.push_back(n);
          A.push_back(ax);
        };
        if (fixed == 2) {
          if (on_bottom || on_top || on_x || on_y)
            for (int8_t ax = 0; ax < 3; ++ax) push(ax);
          continue;
        }
        if (on_bottom) {
          for (int8_t ax = 0; ax < 3; ++ax) push(ax);
          continue;
        }
        if (on_x) push(0);
        if (on_y) push(1);
      }
    }
    for (int u = 0; u < T; ++u) {
      m.bc_node.insert(m.bc_node.end(), bn[u].begin(), bn[u].end());
      m.bc_axis.insert(m.bc_axis.end(), ba[u].begin(), ba[u].end());
    }
  }
  return m;
}

void setup_mark(const char* what) {
  static const bool on = std::getenv("TSGPU_SETUP_PROFILE") != nullptr;
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - last).count());
  last = now;
}

}  // namespace tsg
