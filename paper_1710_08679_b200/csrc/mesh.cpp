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
#include <cstring>

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
  // upper bound of unique edges: 7 per vertex (Kuhn split) -> reserve
  m.coords.reserve(3 * static_cast<size_t>(nv) * 8);
  for (int64_t k = 0; k <= nz; ++k)
    for (int64_t j = 0; j <= ny; ++j)
      for (int64_t i = 0; i <= nx; ++i) {
        m.coords.push_back(i * hx);
        m.coords.push_back(j * hy);
        m.coords.push_back(k * hz);
      }
  static constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                      {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static constexpr int edge_ends[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  const int n_layers = static_cast<int>(interfaces.size()) + 1;
  m.tets10.resize(10 * static_cast<size_t>(ne));
  m.material_id.resize(static_cast<size_t>(ne));
  auto vid = [&](int64_t i, int64_t j, int64_t k) { return i + (nx + 1) * (j + (ny + 1) * k); };
  size_t e = 0;
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i)
        for (const auto& p : perms) {
          int64_t corner[4][3] = {{i, j, k}, {}, {}, {}};
          for (int s = 0; s < 3; ++s) {
            for (int a = 0; a < 3; ++a) corner[s + 1][a] = corner[s][a];
            corner[s + 1][p[s]] += 1;
          }
          int32_t v[4];
          for (int s = 0; s < 4; ++s)
            v[s] = static_cast<int32_t>(vid(corner[s][0], corner[s][1], corner[s][2]));
          const double* c = m.coords.data();
          if (tet_volume(c + 3 * size_t(v[0]), c + 3 * size_t(v[1]), c + 3 * size_t(v[2]),
                         c + 3 * size_t(v[3])) < 0.0)
            std::swap(v[2], v[3]);
          int32_t* t = m.tets10.data() + 10 * e;
          for (int s = 0; s < 4; ++s) t[s] = v[s];
          const double zc = (c[3 * size_t(v[0]) + 2] + c[3 * size_t(v[1]) + 2] +
                             c[3 * size_t(v[2]) + 2] + c[3 * size_t(v[3]) + 2]) / 4.0;
          int below = 0;
          for (double z : interfaces)
            if (zc > z) ++below;
          m.material_id[e] = n_layers - 1 - below;  // layer 0 on top (box_mesh.hpp:75-82)
          ++e;
        }
  // edge midpoints, discovery order; key = lower vertex * 8 + axis-offset bits
  std::vector<int32_t> edge_id(static_cast<size_t>(nv) * 8, -1);
  int32_t nn = static_cast<int32_t>(nv);
  for (size_t q = 0; q < static_cast<size_t>(ne); ++q) {
    int32_t* t = m.tets10.data() + 10 * q;
    for (int s = 0; s < 6; ++s) {
      const int32_t a = t[edge_ends[s][0]], b = t[edge_ends[s][1]];
      const int64_t lo = std::min(a, b), hi = std::max(a, b);
      const int64_t d = hi - lo;  // = di + (nx+1) dj + (nx+1)(ny+1) dk, di,dj,dk in {0,1}
      const int64_t sx = nx + 1, sxy = (nx + 1) * (ny + 1);
      const int64_t dk = d / sxy, dj = (d - dk * sxy) / sx, di = d - dk * sxy - dj * sx;
      const size_t key = static_cast<size_t>(lo) * 8 + size_t(di | (dj << 1) | (dk << 2));
      int32_t id = edge_id[key];
      if (id < 0) {
        id = nn++;
        edge_id[key] = id;
        for (int cc = 0; cc < 3; ++cc)
          m.coords.push_back(0.5 * (m.coords[3 * size_t(a) + cc] + m.coords[3 * size_t(b) + cc]));
      }
      t[4 + s] = id;
    }
  }
  m.coords.shrink_to_fit();
  // Dirichlet set by node coordinate (box_mesh.hpp:134-155)
  if (fixed != 0) {
    const double tol = 1e-9 * std::max({ext[0], ext[1], ext[2]});
    for (int32_t n = 0; n < nn; ++n) {
      const double* c = m.coords.data() + 3 * size_t(n);
      const bool on_bottom = std::abs(c[2]) <= tol;
      const bool on_top = std::abs(c[2] - ext[2]) <= tol;
      const bool on_x = std::abs(c[0]) <= tol || std::abs(c[0] - ext[0]) <= tol;
      const bool on_y = std::abs(c[1]) <= tol || std::abs(c[1] - ext[1]) <= tol;
      auto push = [&](int8_t a) { m.bc_node.push_back(n); m.bc_axis.push_back(a); };
      if (fixed == 2) {
        if (on_bottom || on_top || on_x || on_y)
          for (int8_t a = 0; a < 3; ++a) push(a);
        continue;
      }
      if (on_bottom) {
        for (int8_t a = 0; a < 3; ++a) push(a);
        continue;
      }
      if (on_x) push(0);
      if (on_y) push(1);
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
