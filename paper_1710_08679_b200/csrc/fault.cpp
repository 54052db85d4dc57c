// fault.cpp — host geometry of the Green's-function sweep: fault faces on a
// mesh plane, split nodes, unit slip bases, point location. Restated from the
// reference's fault.hpp / greens.hpp in the same evaluation order (the split
// numbering and the node frames decide the right-hand sides bit for bit).
#include "fault.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <string>
#include <unordered_map>

namespace tsg {
namespace {

V3 add(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
V3 sub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
V3 scl(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
double norm(const V3& a) { return std::sqrt(dot(a, a)); }
V3 normalized(const V3& a) {
  const double n = norm(a);
  return {a[0] / n, a[1] / n, a[2] / n};
}
V3 coord(const Mesh& m, int32_t v) { return {m.coords[3 * size_t(v)], m.coords[3 * size_t(v) + 1], m.coords[3 * size_t(v) + 2]}; }

// face_frame (fault.hpp:122-130)
void face_frame(const V3& a, const V3& b, const V3& c, V3& normal, V3& strike, V3& dip) {
  normal = normalized(cross(sub(b, a), sub(c, a)));
  const V3 up = {0.0, 0.0, 1.0};
  V3 s = cross(up, normal);
  if (norm(s) < 1e-12) s = {1.0, 0.0, 0.0};
  strike = normalized(s);
  dip = cross(strike, normal);
}

constexpr int kFaceVerts[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
constexpr int kEdgeEnds[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};

bool invert3(const double m[3][3], double inv[3][3]) {  // geometry.hpp:27-42
  const double d = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                   m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  if (std::abs(d) <= 0.0 || d == 0.0) return false;
  const double id = 1.0 / d;
  inv[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) * id;
  inv[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * id;
  inv[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * id;
  inv[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) * id;
  inv[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * id;
  inv[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * id;
  inv[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) * id;
  inv[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * id;
  inv[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * id;
  return true;
}

}  // namespace

std::vector<std::array<int32_t, 3>> find_plane_fault_faces(const Mesh& m, int axis, double c0, const V3& lo,
                                                           const V3& hi) {
  if (axis < 0 || axis > 2) validation("fault plane: axis must be 0..2");
  double scale = std::abs(c0);
  for (double x : m.coords) scale = std::max(scale, std::abs(x));
  const double tol = 1e-9 * std::max(scale, 1.0);
  auto on_plane = [&](int32_t v) {
    const V3 c = coord(m, v);
    if (std::abs(c[axis] - c0) > tol) return false;
    for (int a = 0; a < 3; ++a)
      if (c[a] < lo[a] - tol || c[a] > hi[a] + tol) return false;
    return true;
  };
  std::vector<std::array<int32_t, 3>> keys;
  for (int32_t e = 0; e < m.n_elems(); ++e)
    for (const auto& fv : kFaceVerts) {
      std::array<int32_t, 3> key = {m.tets10[10 * size_t(e) + fv[0]], m.tets10[10 * size_t(e) + fv[1]],
                                    m.tets10[10 * size_t(e) + fv[2]]};
      if (!on_plane(key[0]) || !on_plane(key[1]) || !on_plane(key[2])) continue;
      std::sort(key.begin(), key.end());
      keys.push_back(key);
    }
  std::sort(keys.begin(), keys.end());  // the reference's std::map order
  std::vector<std::array<int32_t, 3>> out;
  for (size_t i = 0; i < keys.size();) {
    size_t j = i;
    while (j < keys.size() && keys[j] == keys[i]) ++j;
    if (j - i == 2) out.push_back(keys[i]);
    i = j;
  }
  if (out.empty()) validation("fault plane: no interior faces found on the requested plane");
  return out;
}

void split_nodes(const Mesh& m, const std::vector<std::array<int32_t, 3>>& tris, Mesh& out, FaultPatch& patch) {
  if (tris.empty()) validation("split_nodes: empty fault surface");
  const int32_t V = m.vertex_count, N = m.n_nodes(), E = m.n_elems();
  patch = FaultPatch{};
  std::set<int32_t> fvert, fnode;
  for (const auto& t : tris)
    for (int32_t v : t) {
      if (v < 0 || v >= V) validation("split_nodes: fault vertex " + std::to_string(v) + " is not a mesh vertex");
      fvert.insert(v);
    }
  // edge nodes between fault vertices (the reference's edge_map, mesh.hpp:61-71)
  std::unordered_map<uint64_t, int32_t> emap;
  for (int32_t e = 0; e < E; ++e)
    for (int k = 0; k < 6; ++k) {
      int32_t a = m.tets10[10 * size_t(e) + kEdgeEnds[k][0]], b = m.tets10[10 * size_t(e) + kEdgeEnds[k][1]];
      if (!fvert.count(a) || !fvert.count(b)) continue;
      if (a > b) std::swap(a, b);
      emap[(uint64_t(uint32_t(a)) << 32) | uint32_t(b)] = m.tets10[10 * size_t(e) + 4 + k];
    }
  for (const auto& t : tris) {
    FaultFace f;
    f.verts = t;
    for (int k = 0; k < 3; ++k) {
      int32_t a = t[k], b = t[(k + 1) % 3];
      if (a > b) std::swap(a, b);
      const auto it = emap.find((uint64_t(uint32_t(a)) << 32) | uint32_t(b));
      if (it == emap.end())
        validation("split_nodes: fault triangle edge (" + std::to_string(a) + "," + std::to_string(b) +
                   ") is not a mesh edge");
      f.edges[k] = it->second;
    }
    face_frame(coord(m, t[0]), coord(m, t[1]), coord(m, t[2]), f.normal, f.strike, f.dip);
    patch.faces.push_back(f);
  }
  const V3 ref_normal = patch.faces[0].normal;
  for (auto& f : patch.faces)
    if (dot(f.normal, ref_normal) < 0.0) {
      std::swap(f.verts[1], f.verts[2]);
      face_frame(coord(m, f.verts[0]), coord(m, f.verts[1]), coord(m, f.verts[2]), f.normal, f.strike, f.dip);
    }
  for (const auto& f : patch.faces) {
    for (int32_t v : f.verts) fnode.insert(v);
    for (int32_t e : f.edges) fnode.insert(e);
  }
  for (size_t i = 0; i < m.bc_node.size(); ++i)
    if (fnode.count(m.bc_node[i]))
      validation("split_nodes: fault face adjacent to a Dirichlet boundary (node " + std::to_string(m.bc_node[i]) +
                 ")");
  {
    std::map<std::array<int32_t, 3>, int> face_elems;
    for (int32_t e = 0; e < E; ++e)
      for (const auto& fv : kFaceVerts) {
        std::array<int32_t, 3> key = {m.tets10[10 * size_t(e) + fv[0]], m.tets10[10 * size_t(e) + fv[1]],
                                      m.tets10[10 * size_t(e) + fv[2]]};
        std::sort(key.begin(), key.end());
        if (!fvert.count(key[0]) || !fvert.count(key[1]) || !fvert.count(key[2])) continue;
        ++face_elems[key];
      }
    for (const auto& f : patch.faces) {
      std::array<int32_t, 3> key = f.verts;
      std::sort(key.begin(), key.end());
      const auto it = face_elems.find(key);
      if (it == face_elems.end() || it->second != 2)
        validation("split_nodes: fault face (" + std::to_string(f.verts[0]) + "," + std::to_string(f.verts[1]) +
                   "," + std::to_string(f.verts[2]) + ") is not an interior manifold face");
    }
  }
  const double plane_d = dot(ref_normal, coord(m, patch.faces[0].verts[0]));
  std::map<int32_t, V3> node_strike, node_dip;
  for (const auto& f : patch.faces)
    for (int k = 0; k < 3; ++k)
      for (int32_t nd : {f.verts[k], f.edges[k]}) {
        V3& s = node_strike[nd];
        V3& d = node_dip[nd];
        s = add(s, f.strike);
        d = add(d, f.dip);
      }
  std::vector<int8_t> side(E, 0);
  for (int32_t e = 0; e < E; ++e) {
    bool touches = false;
    for (int k = 0; k < 10 && !touches; ++k) touches = fnode.count(m.tets10[10 * size_t(e) + k]) != 0;
    if (!touches) continue;
    V3 c = {0, 0, 0};
    for (int k = 0; k < 4; ++k) c = add(c, coord(m, m.tets10[10 * size_t(e) + k]));
    c = scl(0.25, c);
    const double s = dot(ref_normal, c) - plane_d;
    if (s == 0.0)
      validation("split_nodes: element " + std::to_string(e) + " centroid lies on the fault plane; cannot classify side");
    side[e] = s > 0.0 ? int8_t(1) : int8_t(-1);
  }
  std::vector<int32_t> dup_v, dup_e;
  for (int32_t nd : fnode) (nd < V ? dup_v : dup_e).push_back(nd);
  const int32_t ndv = static_cast<int32_t>(dup_v.size());
  auto renum = [&](int32_t old) { return old < V ? old : old + ndv; };
  std::map<int32_t, int32_t> plus_of;
  for (size_t i = 0; i < dup_v.size(); ++i) plus_of[dup_v[i]] = V + static_cast<int32_t>(i);
  for (size_t i = 0; i < dup_e.size(); ++i) plus_of[dup_e[i]] = N + ndv + static_cast<int32_t>(i);
  out = Mesh{};
  out.vertex_count = V + ndv;
  const int32_t NS = N + ndv + static_cast<int32_t>(dup_e.size());
  out.coords.assign(3 * size_t(NS), 0.0);
  patch.to_base.assign(NS, -1);
  for (int32_t nd = 0; nd < N; ++nd) {
    for (int c = 0; c < 3; ++c) out.coords[3 * size_t(renum(nd)) + c] = m.coords[3 * size_t(nd) + c];
    patch.to_base[renum(nd)] = nd;
  }
  for (const auto& [base, plus] : plus_of) {
    for (int c = 0; c < 3; ++c) out.coords[3 * size_t(plus) + c] = m.coords[3 * size_t(base) + c];
    patch.to_base[plus] = base;
  }
  out.tets10.resize(m.tets10.size());
  out.material_id = m.material_id;
  for (int32_t e = 0; e < E; ++e)
    for (int k = 0; k < 10; ++k) {
      const int32_t old = m.tets10[10 * size_t(e) + k];
      int32_t nid = renum(old);
      if (side[e] > 0 && fnode.count(old)) nid = plus_of[old];
      out.tets10[10 * size_t(e) + k] = nid;
    }
  for (size_t i = 0; i < m.bc_node.size(); ++i) {
    out.bc_node.push_back(renum(m.bc_node[i]));
    out.bc_axis.push_back(m.bc_axis[i]);
  }
  patch.split_nodes.reserve(fnode.size());
  for (int32_t base : fnode) {
    SplitNode sn;
    sn.base = base;
    sn.minus = renum(base);
    sn.plus = plus_of[base];
    sn.coord = coord(m, base);
    sn.strike = normalized(node_strike[base]);
    sn.dip = normalized(node_dip[base]);
    patch.split_nodes.push_back(sn);
  }
}

double bspline_bell(double s) {
  const double t = 1.5 * std::abs(s);
  double v = 0.0;
  if (t <= 0.5) v = 0.75 - t * t;
  else if (t <= 1.5) v = 0.5 * (1.5 - t) * (1.5 - t);
  return v / 0.75;
}

std::vector<double> unit_slip_magnitudes(const FaultPatch& patch, const Mesh& base, const V3& center, double radius) {
  if (radius <= 0.0) validation("unit_slip_basis: radius must be positive");
  if (patch.faces.empty()) validation("unit_slip_basis: empty fault patch");
  const V3& n = patch.faces[0].normal;
  const V3 p0 = coord(base, patch.faces[0].verts[0]);
  const double scale = std::max(radius, norm(sub(center, p0)));
  if (std::abs(dot(sub(center, p0), n)) > 1e-6 * scale)
    validation("unit_slip_basis: center does not lie on the fault plane");
  std::vector<double> mag(patch.split_nodes.size());
  for (size_t i = 0; i < mag.size(); ++i) mag[i] = bspline_bell(norm(sub(patch.split_nodes[i].coord, center)) / radius);
  return mag;
}

// tet10_shape_values (element_stiffness.hpp:56-61) of element e at point p
void tet10_shape_at(const Mesh& m, int32_t e, const V3& p, double n10[10]) {
  const V3 v0 = coord(m, m.tets10[10 * size_t(e)]);
  double jac[3][3], inv[3][3];
  for (int c = 0; c < 3; ++c) {
    const V3 ed = sub(coord(m, m.tets10[10 * size_t(e) + c + 1]), v0);
    for (int r = 0; r < 3; ++r) jac[r][c] = ed[r];
  }
  invert3(jac, inv);
  const V3 d = sub(p, v0);
  double xi[3];
  for (int r = 0; r < 3; ++r) xi[r] = inv[r][0] * d[0] + inv[r][1] * d[1] + inv[r][2] * d[2];
  const double l[4] = {1.0 - xi[0] - xi[1] - xi[2], xi[0], xi[1], xi[2]};
  for (int a = 0; a < 4; ++a) n10[a] = l[a] * (2.0 * l[a] - 1.0);
  for (int k = 0; k < 6; ++k) n10[4 + k] = 4.0 * l[kEdgeEnds[k][0]] * l[kEdgeEnds[k][1]];
}

}  // namespace tsg
