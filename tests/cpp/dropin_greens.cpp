// A Green's-function sweep written against the reference's API (fault.hpp, model.hpp, greens.hpp):
// only the include differs. Prints one JSON line for tests/test_dropin_cpp.py to compare with the
// reference itself.
#include <cstdio>
#include <vector>

#include "tetsolve_b200/tetsolve.hpp"

using namespace tetsolve;

int main() {
  BoxMeshSpec spec;
  spec.extents = {8000.0, 8000.0, 6000.0};
  spec.divisions = {8, 8, 6};
  spec.layer_interfaces = {4500.0};
  Mesh mesh = generate_box_mesh(spec);
  const std::vector<Material> mats = {material_from_wavespeeds(1600, 400, 1850),
                                      material_from_wavespeeds(5800, 3000, 2700)};
  const auto faces = find_plane_fault_faces(mesh, 0, 4000.0, {4000.0, 2000.0, 1000.0}, {4000.0, 6000.0, 5000.0});
  SolverConfig cfg;
  cfg.batch_size = 2;
  const FaultedModel fm = build_faulted_model(mesh, mats, faces, cfg);
  const Vec3 centers[5] = {{4000.0, 4000.0, 3000.0}, {4000.0, 3000.0, 2500.0}, {4000.0, 5000.0, 4000.0},
                           {4000.0, 4000.0, 3000.0}, {4000.0, 3500.0, 2000.0}};
  const SlipDirection dirs[5] = {SlipDirection::dip, SlipDirection::dip, SlipDirection::strike,
                                 SlipDirection::strike, SlipDirection::dip};
  const double radii[5] = {1500.0, 1000.0, 1200.0, 1500.0, 900.0};
  std::vector<UnitSlip> slips;
  for (int i = 0; i < 5; ++i) slips.push_back(unit_slip_basis(fm.patch, fm.base.mesh, centers[i], dirs[i], radii[i]));
  const Vec3 pts[6] = {{1000.0, 2000.0, 6000.0}, {3000.0, 4000.0, 6000.0}, {5000.0, 4000.0, 6000.0},
                       {6500.0, 1500.0, 6000.0}, {4000.0, 7000.0, 6000.0}, {2500.0, 2500.0, 5500.0}};
  const int axes[6] = {0, 1, 2, 0, 2, 1};
  std::vector<ObservationComponent> obs;
  for (int r = 0; r < 6; ++r) obs.push_back({pts[r], axes[r]});
  const auto [bank, rep] = compute_greens_bank(fm, slips, obs, cfg);
  // the reference's file formats round-trip the sweep's inputs and outputs
  write_fault_faces(faces, "dropin_greens.tsfault");
  write_greens_bank(bank, "dropin_greens.tsgreens");
  const bool files_ok = read_fault_faces("dropin_greens.tsfault") == faces &&
                        read_greens_bank("dropin_greens.tsgreens").values == bank.values;
  std::remove("dropin_greens.tsfault");
  std::remove("dropin_greens.tsgreens");
  const VectorBatch64 f0 = slip_to_rhs(fm, slips[0]);
  double f0n = 0.0;
  for (double x : f0.data) f0n += x * x;
  // the base level set is usable directly: solve one right-hand side
  VectorBatch64 u0(fm.base.mesh.node_count(), 1);
  SolverConfig c1 = cfg;
  c1.batch_size = 1;
  const auto sol = solve(fm.base.levels, f0, u0, c1);
  std::printf("{\"faces\": %zu, \"split_nodes\": %d, \"split_mesh_nodes\": %d, \"calls\": %d, \"outer\": %ld, "
              "\"f0_norm2\": %.17g, \"solve_outer\": %d, \"files_ok\": %d, \"bank\": [",
              faces.size(), fm.patch.n_split_nodes, fm.split_mesh_nodes, rep.solver_calls, rep.outer_iterations, f0n,
              sol.second.outer_iterations, files_ok ? 1 : 0);
  for (size_t i = 0; i < bank.values.size(); ++i) std::printf("%s%.17g", i ? ", " : "", bank.values[i]);
  std::printf("]}\n");
  return 0;
}
