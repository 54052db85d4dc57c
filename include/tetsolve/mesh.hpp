// tetsolve/mesh.hpp — drop-in for mesh.hpp:19-156: the host Mesh value type
// (vertices first, tets10 = 4 vertices + 6 edge nodes on edges
// (0,1),(1,2),(2,0),(0,3),(1,3),(2,3)) and its checks. validate_mesh runs the
// library's validator (the reference's checks and messages, parallel).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "tetsolve/errors.hpp"
#include "tetsolve/geometry.hpp"

namespace tetsolve {

struct DirichletBc {  // mesh.hpp:19-23
  int32_t node = 0;
  int8_t axis = 0;
  friend bool operator==(const DirichletBc&, const DirichletBc&) = default;
};

struct Mesh {  // mesh.hpp:26-42
  std::vector<Vec3> coords;
  std::vector<std::array<int32_t, 10>> tets10;
  std::vector<std::array<int32_t, 4>> tets4;
  std::vector<int32_t> material_id;
  std::map<std::pair<int32_t, int32_t>, int32_t> edge_map;
  int32_t vertex_count = 0;
  std::vector<DirichletBc> dirichlet;
  int32_t node_count() const { return static_cast<int32_t>(coords.size()); }
  int32_t element_count() const { return static_cast<int32_t>(tets10.size()); }
  double element_volume(int32_t e) const {
    const auto& t = tets4[e];
    return tet_volume(coords[t[0]], coords[t[1]], coords[t[2]], coords[t[3]]);
  }
};

struct P1View {  // mesh.hpp:46-57
  const Mesh* parent = nullptr;
  int32_t node_count = 0;
  const std::vector<std::array<int32_t, 4>>* tets4 = nullptr;
};
inline P1View p1_restrict_view(const Mesh& m) { return P1View{&m, m.vertex_count, &m.tets4}; }
inline P1View p1_restrict_view(const P1View& v) { return v; }

// rebuild_edge_map (mesh.hpp:61-71)
inline void rebuild_edge_map(Mesh& m) {
  static constexpr int ee[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  m.edge_map.clear();
  for (const auto& t : m.tets10)
    for (int k = 0; k < 6; ++k) {
      int32_t a = t[ee[k][0]], b = t[ee[k][1]];
      if (a > b) std::swap(a, b);
      m.edge_map[{a, b}] = t[4 + k];
    }
}

// dirichlet_mask (mesh.hpp:150-154)
inline std::vector<uint8_t> dirichlet_mask(const Mesh& m) {
  std::vector<uint8_t> mask(3 * static_cast<size_t>(m.node_count()), 0);
  for (const auto& bc : m.dirichlet) mask[3 * static_cast<size_t>(bc.node) + bc.axis] = 1;
  return mask;
}

namespace detail {
// the library's copy of a Mesh (ts_mesh): coords, tets10, material ids, Dirichlet list
struct MeshHandle {
  ts_mesh* h = nullptr;
  explicit MeshHandle(const Mesh& m) {
    if (m.material_id.size() != m.tets10.size() || (!m.tets4.empty() && m.tets4.size() != m.tets10.size()))
      throw ValidationError("mesh: inconsistent per-element array sizes");
    for (size_t e = 0; e < m.tets4.size(); ++e)
      for (int k = 0; k < 4; ++k)
        if (m.tets4[e][k] != m.tets10[e][k])
          throw ValidationError("mesh: element " + std::to_string(e) + ": tets4 is not the vertex prefix of tets10");
    std::vector<double> c(3 * m.coords.size());
    for (size_t i = 0; i < m.coords.size(); ++i)
      for (int k = 0; k < 3; ++k) c[3 * i + k] = m.coords[i][k];
    std::vector<int32_t> t(10 * m.tets10.size());
    for (size_t e = 0; e < m.tets10.size(); ++e)
      for (int a = 0; a < 10; ++a) t[10 * e + a] = m.tets10[e][a];
    std::vector<int32_t> bn(m.dirichlet.size());
    std::vector<int8_t> ba(m.dirichlet.size());
    for (size_t i = 0; i < m.dirichlet.size(); ++i) {
      bn[i] = m.dirichlet[i].node;
      ba[i] = m.dirichlet[i].axis;
    }
    check(ts_mesh_from_arrays(m.node_count(), m.vertex_count, c.data(), m.element_count(), t.data(),
                              m.material_id.data(), static_cast<int32_t>(bn.size()), bn.data(), ba.data(), &h));
  }
  ~MeshHandle() { ts_mesh_destroy(h); }
  MeshHandle(const MeshHandle&) = delete;
  MeshHandle& operator=(const MeshHandle&) = delete;
};

// a library mesh handle as the reference's Mesh (edge_map rebuilt as rebuild_edge_map)
inline Mesh take_mesh(ts_mesh* h) {
  int32_t nn, nv, ne, nbc;
  ts_mesh_sizes(h, &nn, &nv, &ne, &nbc);
  std::vector<double> c(3 * size_t(nn));
  std::vector<int32_t> t(10 * size_t(ne)), mat(ne), bn(nbc);
  std::vector<int8_t> ba(nbc);
  ts_mesh_export(h, c.data(), t.data(), mat.data(), bn.data(), ba.data());
  ts_mesh_destroy(h);
  Mesh m;
  m.vertex_count = nv;
  m.coords.resize(nn);
  for (int32_t i = 0; i < nn; ++i) m.coords[i] = {c[3 * size_t(i)], c[3 * size_t(i) + 1], c[3 * size_t(i) + 2]};
  m.tets10.resize(ne);
  m.tets4.resize(ne);
  for (int32_t e = 0; e < ne; ++e) {
    for (int a = 0; a < 10; ++a) m.tets10[e][a] = t[10 * size_t(e) + a];
    for (int a = 0; a < 4; ++a) m.tets4[e][a] = t[10 * size_t(e) + a];
  }
  rebuild_edge_map(m);
  m.material_id = std::move(mat);
  for (int32_t i = 0; i < nbc; ++i) m.dirichlet.push_back({bn[i], ba[i]});
  return m;
}
}  // namespace detail

// validate_mesh (mesh.hpp:75-113): ValidationError naming the first offending element or node
inline void validate_mesh(const Mesh& m) {
  if (m.vertex_count < 0 || m.vertex_count > m.node_count()) throw ValidationError("mesh: vertex_count out of range");
  if (m.tets4.size() != m.tets10.size() || m.material_id.size() != m.tets10.size())
    throw ValidationError("mesh: inconsistent per-element array sizes");
  detail::MeshHandle h(m);
  detail::check(ts_mesh_validate(h.h));
}

inline double total_volume(const Mesh& m) {  // mesh.hpp:116-120
  double v = 0.0;
  for (int32_t e = 0; e < m.element_count(); ++e) v += m.element_volume(e);
  return v;
}

struct FaceCensus {  // mesh.hpp:124-128
  int64_t interior = 0;
  int64_t boundary = 0;
  int max_share = 0;
};
// count_faces (mesh.hpp:130-147): topology census (integer bookkeeping, host)
inline FaceCensus count_faces(const Mesh& m) {
  std::map<std::array<int32_t, 3>, int> faces;
  static constexpr int fv[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
  for (const auto& t : m.tets4)
    for (const auto& f : fv) {
      std::array<int32_t, 3> key = {t[f[0]], t[f[1]], t[f[2]]};
      std::sort(key.begin(), key.end());
      ++faces[key];
    }
  FaceCensus c;
  for (const auto& kv : faces) {
    if (kv.second == 1) ++c.boundary;
    else if (kv.second == 2) ++c.interior;
    c.max_share = std::max(c.max_share, kv.second);
  }
  return c;
}

}  // namespace tetsolve
