// Drop-in demo: the reference's manufactured-solution test (test_solver.cpp:137-181)
// written against tetsolve_b200/tetsolve.hpp instead of the reference headers.
// Build: g++ -std=c++20 -Iinclude tests/cpp/dropin_demo.cpp -Lpaper_1710_08679_b200 -ltsgpu
#include <cmath>
#include <cstdio>

#include "tetsolve_b200/tetsolve.hpp"

using namespace tetsolve;

int main() {
  const Vec3 ext = {400.0, 400.0, 200.0};
  BoxMeshSpec spec;
  spec.extents = ext;
  spec.divisions = {4, 4, 4};
  spec.layer_interfaces = {100.0};
  Mesh mesh = generate_box_mesh(spec);
  const std::vector<Material> mats = {material_from_wavespeeds(1600.0, 400.0, 1850.0),
                                      material_from_wavespeeds(5800.0, 3000.0, 2700.0)};
  SolverConfig cfg;
  cfg.batch_size = 2;
  const CrustModel model = build_crust_model(mesh, mats, cfg);
  const double pi = 3.14159265358979323846;
  VectorBatch64 ustar(model.mesh.node_count(), 2);
  for (int32_t n = 0; n < model.mesh.node_count(); ++n) {
    const Vec3& x = model.mesh.coords[n];
    const double sx = std::sin(pi * x[0] / ext[0]), cx = std::cos(pi * x[0] / ext[0]);
    const double sy = std::sin(pi * x[1] / ext[1]), cy = std::cos(pi * x[1] / ext[1]);
    const double sz = std::sin(0.5 * pi * x[2] / ext[2]);
    const double v[3] = {0.05 * sx * cy * sz, 0.05 * cx * sy * sz, 0.05 * cx * cy * sz};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 2; ++b) ustar.at(3 * int64_t(n) + a, b) = model.mask[3 * size_t(n) + a] ? 0.0 : v[a];
  }
  VectorBatch64 f;
  model.levels.outer.apply(ustar, f);
  VectorBatch64 u0(model.mesh.node_count(), 2);
  auto [u, rep] = solve(model.levels, f, u0, cfg);
  double num = 0, den = 0;
  for (size_t i = 0; i < u.data.size(); ++i) {
    num += (u.data[i] - ustar.data[i]) * (u.data[i] - ustar.data[i]);
    den += ustar.data[i] * ustar.data[i];
  }
  auto [up, repp] = solve_pcge(model.levels.outer, f, u0, 1e-8, 100000);
  bool threw = false;
  try {
    VectorBatch64 bad(model.mesh.node_count() + 1, 1), out;
    model.levels.outer.apply(bad, out);
  } catch (const ValidationError&) {
    threw = true;
  }
  std::printf("{\"converged\": %d, \"outer\": %d, \"inner\": [%ld, %ld, %ld], \"max_final\": %.3e, "
              "\"rel_err\": %.3e, \"history\": %zu, \"pcge_outer\": %d, \"method\": \"%s\", \"validation_throw\": %d}\n",
              rep.converged, rep.outer_iterations, rep.inner_iterations[0], rep.inner_iterations[1],
              rep.inner_iterations[2], rep.max_final_residual(), std::sqrt(num / den), rep.residual_history.size(),
              repp.outer_iterations, repp.method.c_str(), threw);
  return rep.converged && std::sqrt(num / den) < 1e-7 && threw ? 0 : 1;
}
