// tetsolve/model.hpp — drop-in for model.hpp:14-58: CrustModel and the
// faulted model of the Green's-function sweep.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "tetsolve/adaptive_cg.hpp"
#include "tetsolve/fault.hpp"
#include "tetsolve/material.hpp"
#include "tetsolve/mesh.hpp"

namespace tetsolve {

struct CrustModel {  // model.hpp:14-19
  Mesh mesh;
  std::vector<Material> materials;
  std::vector<uint8_t> mask;
  SolverLevels levels;
};

// build_crust_model (model.hpp:21-29)
inline CrustModel build_crust_model(Mesh mesh, std::vector<Material> materials, const SolverConfig& cfg,
                                    int workers = 1) {
  CrustModel model;
  model.mask = dirichlet_mask(mesh);
  model.levels = build_solver_levels(mesh, materials, model.mask, cfg, workers);
  model.mesh = std::move(mesh);
  model.materials = std::move(materials);
  return model;
}

struct FaultedModel {  // model.hpp:34-39 (split mesh and raw split operator live in the library)
  CrustModel base;
  FaultPatch patch;
  int32_t split_mesh_nodes = 0;
  std::shared_ptr<ts_faulted> handle;
};

// build_faulted_model (model.hpp:41-51)
inline FaultedModel build_faulted_model(Mesh mesh, std::vector<Material> materials,
                                        const std::vector<std::array<int32_t, 3>>& fault_tris,
                                        const SolverConfig& cfg, int /*workers*/ = 1) {
  detail::MeshHandle h(mesh);
  const auto [lam, mu] = detail::lame(materials);
  const ts_solver_config c = cfg.to_c();
  ts_faulted* f = nullptr;
  detail::check(ts_faulted_model_create(h.h, static_cast<int32_t>(materials.size()), lam.data(), mu.data(),
                                        fault_tris.empty() ? nullptr : fault_tris[0].data(),
                                        static_cast<int32_t>(fault_tris.size()), &c, &f));
  FaultedModel fm;
  fm.handle = std::shared_ptr<ts_faulted>(f, ts_faulted_model_destroy);
  detail::check(ts_faulted_info(f, &fm.patch.n_split_nodes, &fm.split_mesh_nodes, &fm.patch.n_faces));
  ts_levels* lv = nullptr;
  detail::check(ts_faulted_levels(f, &lv));
  fm.base.mask = dirichlet_mask(mesh);
  fm.base.levels = SolverLevels(std::shared_ptr<ts_levels>(fm.handle, lv), mesh);
  fm.base.mesh = std::move(mesh);
  fm.base.materials = std::move(materials);
  return fm;
}

namespace detail {
struct SlipArrays {
  std::vector<double> centers, radii;
  std::vector<int32_t> dirs;
  explicit SlipArrays(const std::vector<UnitSlip>& slips) {
    for (const auto& s : slips) {
      centers.insert(centers.end(), s.center.begin(), s.center.end());
      dirs.push_back(static_cast<int32_t>(s.direction));
      radii.push_back(s.radius);
    }
  }
};
}  // namespace detail

// slip_to_rhs (model.hpp:53-56): one fp64 EBE product on the split mesh
inline VectorBatch64 slip_to_rhs(const FaultedModel& fm, const UnitSlip& slip) {
  const detail::SlipArrays a({slip});
  VectorBatch64 f(fm.base.mesh.node_count(), 1);
  detail::check(ts_slip_to_rhs(fm.handle.get(), 1, a.centers.data(), a.dirs.data(), a.radii.data(), f.data.data()));
  return f;
}

}  // namespace tetsolve
