// tetsolve/fault.hpp — drop-in for the fault.hpp types and entry points a
// Green's-function sweep uses (fault.hpp:12-421): split-node geometry, unit
// slip bases and slip lifting run inside the library (csrc/fault.cpp,
// csrc/greens.cu); FaultPatch is a summary (its geometry stays there) and
// UnitSlip magnitudes are evaluated there.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "tetsolve/mesh.hpp"

namespace tetsolve {

enum class SlipDirection { dip = 0, strike = 1 };  // fault.hpp:12-15

struct FaultPatch {  // fault.hpp:37-41 (summary)
  int32_t n_faces = 0;
  int32_t n_split_nodes = 0;
};

struct UnitSlip {  // fault.hpp:308-315
  Vec3 center{};
  SlipDirection direction = SlipDirection::dip;
  double radius = 0.0;
  std::vector<double> magnitude;  // evaluated by the library
};

// find_plane_fault_faces (fault.hpp:86-118)
inline std::vector<std::array<int32_t, 3>> find_plane_fault_faces(const Mesh& mesh, int axis, double coord,
                                                                  const Vec3& lo, const Vec3& hi) {
  detail::MeshHandle h(mesh);
  int32_t n = 0;
  detail::check(ts_fault_plane_faces(h.h, axis, coord, lo.data(), hi.data(), &n, nullptr));
  std::vector<std::array<int32_t, 3>> faces(n);
  if (n) detail::check(ts_fault_plane_faces(h.h, axis, coord, lo.data(), hi.data(), &n, faces[0].data()));
  return faces;
}

// unit_slip_basis (fault.hpp:325-343)
inline UnitSlip unit_slip_basis(const FaultPatch& patch, const Mesh& /*base_mesh*/, const Vec3& center,
                                SlipDirection direction, double radius) {
  if (radius <= 0.0) throw ValidationError("unit_slip_basis: radius must be positive");
  if (patch.n_faces == 0) throw ValidationError("unit_slip_basis: empty fault patch");
  UnitSlip s;
  s.center = center;
  s.direction = direction;
  s.radius = radius;
  return s;
}

// TSFAULT 1 fault-face files (fault.hpp:44-84, 414-419): the reference's bytes
inline void write_fault_faces(const std::vector<std::array<int32_t, 3>>& faces, const std::string& path) {
  detail::check(ts_fault_faces_write(path.c_str(), faces.empty() ? nullptr : faces[0].data(),
                                     static_cast<int32_t>(faces.size())));
}
inline std::vector<std::array<int32_t, 3>> read_fault_faces(const std::string& path) {
  int32_t n = 0;
  detail::check(ts_fault_faces_read(path.c_str(), &n, nullptr));
  std::vector<std::array<int32_t, 3>> f(n);
  detail::check(ts_fault_faces_read(path.c_str(), &n, f.empty() ? nullptr : f[0].data()));
  return f;
}

}  // namespace tetsolve
