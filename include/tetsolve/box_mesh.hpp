// tetsolve/box_mesh.hpp — drop-in for box_mesh.hpp:13-157 (layered box
// generator; the library's parallel generator numbers nodes identically).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "tetsolve/mesh.hpp"

namespace tetsolve {

enum class FixedBoundary { none, bottom_and_sides, all_clamped };  // box_mesh.hpp:13-17

struct BoxMeshSpec {  // box_mesh.hpp:23-28
  Vec3 extents = {1.0, 1.0, 1.0};
  std::array<int32_t, 3> divisions = {1, 1, 1};
  std::vector<double> layer_interfaces;
  FixedBoundary fixed_boundary = FixedBoundary::bottom_and_sides;
};

// generate_box_mesh (box_mesh.hpp:55-157)
inline Mesh generate_box_mesh(const BoxMeshSpec& spec) {
  ts_mesh* h = nullptr;
  detail::check(ts_box_mesh(spec.extents.data(), spec.divisions.data(),
                            static_cast<int32_t>(spec.layer_interfaces.size()), spec.layer_interfaces.data(),
                            static_cast<int32_t>(spec.fixed_boundary), &h));
  return detail::take_mesh(h);
}

}  // namespace tetsolve
