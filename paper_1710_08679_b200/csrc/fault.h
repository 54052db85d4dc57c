// fault.h — the Green's-function sweep around the solve:
// split-node fault surfaces (fault.hpp:86-302), unit slip bases
// (fault.hpp:317-361), slip lifting (fault.hpp:363-388) and surface sampling
// (greens.hpp:50-76) inside the batched bank loop (greens.hpp:114-145).
// Host-side geometry; the products, solves and sampling run on the device.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "ts_common.h"

namespace tsg {

using V3 = std::array<double, 3>;

struct FaultFace {  // fault.hpp:16-21
  std::array<int32_t, 3> verts{}, edges{};
  V3 normal{}, strike{}, dip{};
};
struct SplitNode {  // fault.hpp:25-30
  int32_t base = 0, minus = 0, plus = 0;
  V3 coord{}, strike{}, dip{};
};
struct FaultPatch {  // fault.hpp:32-36
  std::vector<FaultFace> faces;
  std::vector<SplitNode> split_nodes;
  std::vector<int32_t> to_base;
};

// find_plane_fault_faces (fault.hpp:86-118): interior triangles on {axis = coord} inside [lo, hi]
std::vector<std::array<int32_t, 3>> find_plane_fault_faces(const Mesh& m, int axis, double coord, const V3& lo,
                                                           const V3& hi);
// split_nodes (fault.hpp:140-302): duplicated fault nodes, plus-side elements renumbered
void split_nodes(const Mesh& m, const std::vector<std::array<int32_t, 3>>& tris, Mesh& split, FaultPatch& patch);
// quadratic B-spline bell (fault.hpp:317-323) and unit_slip_basis magnitudes (fault.hpp:325-343)
double bspline_bell(double s);
std::vector<double> unit_slip_magnitudes(const FaultPatch& patch, const Mesh& base, const V3& center,
                                         double radius);
// sample_displacement (greens.hpp:50-76): tet10 shape values of element e at p. The first
// containing element itself is found on the device (greens.cu locate_points).
void tet10_shape_at(const Mesh& m, int32_t e, const V3& p, double n10[10]);

}  // namespace tsg
