// tetsolve/adaptive_cg.hpp — drop-in for adaptive_cg.hpp:20-281: the level
// hierarchy and the solvers. SolverLevels keeps the reference's public
// members (adaptive_cg.hpp:27-37) as host snapshots of the device hierarchy;
// solve / solve_pcge run entirely on the GPU (ts_solve, ts_solve_pcge): H2D
// of f and u0 on entry, D2H of u on exit.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "tetsolve/aggregation.hpp"
#include "tetsolve/block_csr.hpp"
#include "tetsolve/block_jacobi.hpp"
#include "tetsolve/ebe_operator.hpp"
#include "tetsolve/material.hpp"
#include "tetsolve/mesh.hpp"
#include "tetsolve/pcg.hpp"
#include "tetsolve/prolongation.hpp"
#include "tetsolve/solver_config.hpp"
#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

class SolverLevels {  // adaptive_cg.hpp:27-37
 public:
  SolverLevels() = default;
  // the level set `lv` (owned by the shared pointer, possibly through a faulted model) of `mesh`
  SolverLevels(std::shared_ptr<ts_levels> lv, const Mesh& mesh) : lv_(std::move(lv)) {
    ts_levels* h = lv_.get();
    int32_t n0 = 0, n1 = 0, n2 = 0;
    int64_t nnzb2 = 0;
    detail::check(ts_levels_sizes(h, &n0, &n1, &n2, &nnzb2));
    const int32_t ne = mesh.element_count();
    auto conn10 = std::make_shared<std::vector<int32_t>>(10 * size_t(ne));
    auto conn4 = std::make_shared<std::vector<int32_t>>(4 * size_t(ne));
    for (int32_t e = 0; e < ne; ++e) {
      for (int a = 0; a < 10; ++a) (*conn10)[10 * size_t(e) + a] = mesh.tets10[e][a];
      for (int a = 0; a < 4; ++a) (*conn4)[4 * size_t(e) + a] = mesh.tets10[e][a];
    }
    mask0.resize(3 * size_t(n0));
    mask1.resize(3 * size_t(n1));
    mask2.resize(3 * size_t(n2));
    m0.inv_blocks.resize(n0);
    m1.inv_blocks.resize(n1);
    m2.inv_blocks.resize(n2);
    aggregation.agg_of_node.resize(n1);
    aggregation.n_aggregates = n2;
    aggregation.seeds.resize(n2);
    level2.n_block_rows = n2;
    level2.row_ptr.resize(size_t(n2) + 1);
    level2.col_idx.resize(nnzb2);
    level2.blocks.resize(nnzb2);
    detail::check(ts_levels_export(h, aggregation.agg_of_node.data(), level2.row_ptr.data(), level2.col_idx.data(),
                                   nnzb2 ? level2.blocks[0].data() : nullptr, mask2.data(),
                                   n2 ? m2.inv_blocks[0].data() : nullptr));
    detail::check(ts_levels_export_fine(h, n0 ? m0.inv_blocks[0].data() : nullptr,
                                        n1 ? m1.inv_blocks[0].data() : nullptr, mask0.data(), mask1.data(),
                                        aggregation.seeds.data()));
    auto keep = lv_;
    auto view = [&](int which) {
      const ts_ebe* p = nullptr;
      detail::check(ts_levels_operator(h, which, &p));
      return std::shared_ptr<ts_ebe>(keep, const_cast<ts_ebe*>(p));
    };
    outer = EbeOperator<double>(view(0), n0, ne, 2, conn10, mask0);
    level0 = EbeOperator<float>(view(1), n0, ne, 2, conn10, mask0);
    level1 = EbeOperator<float>(view(2), n1, ne, 1, conn4, mask1);
    p1 = build_geometric_prolongation(mesh);
    p2.kind = Prolongation::Kind::aggregation_l2_to_l1;
    p2.n_fine_nodes = n1;
    p2.n_coarse_nodes = n2;
    p2.row_ptr.resize(size_t(n1) + 1);
    for (int32_t i = 0; i <= n1; ++i) p2.row_ptr[i] = i;
    p2.cols = aggregation.agg_of_node;
    p2.weights.assign(n1, 1.0);
  }

  EbeOperator<double> outer;     // 64-bit second-order EBE (outer loop)
  EbeOperator<float> level0;     // 32-bit second-order EBE
  EbeOperator<float> level1;     // 32-bit first-order EBE
  BlockCsrMatrix<float> level2;  // 32-bit Galerkin coarse matrix
  Prolongation p1;               // level 1 -> level 0 (geometric)
  Prolongation p2;               // level 2 -> level 1 (aggregation)
  BlockJacobi<float> m0, m1, m2;
  std::vector<uint8_t> mask0, mask1, mask2;
  Aggregation aggregation;

  ts_levels* handle() const { return lv_.get(); }

 private:
  std::shared_ptr<ts_levels> lv_;
};

// build_solver_levels (adaptive_cg.hpp:39-67): setup on the host (the reference's
// sequential aggregation, bit-exact) and the device (operators, block Jacobi)
inline SolverLevels build_solver_levels(const Mesh& mesh, const std::vector<Material>& materials,
                                        const std::vector<uint8_t>& dof_mask, const SolverConfig& cfg,
                                        int workers = 1) {
  (void)workers;
  cfg.validate();
  detail::MeshHandle mh(mesh);
  auto [l, m] = detail::lame(materials);
  const ts_solver_config c = cfg.to_c();
  ts_levels* h = nullptr;
  detail::check(ts_levels_create(mh.h, static_cast<int32_t>(l.size()), l.data(), m.data(),
                                 dof_mask.empty() ? nullptr : dof_mask.data(), &c, &h));
  return SolverLevels(std::shared_ptr<ts_levels>(h, ts_levels_destroy), mesh);
}

// solve (adaptive_cg.hpp:242-263)
inline std::pair<VectorBatch64, SolveReport> solve(const SolverLevels& levels, const VectorBatch64& f,
                                                   const VectorBatch64& u0, const SolverConfig& cfg) {
  cfg.validate();
  if (f.n_nodes != levels.outer.n_nodes()) throw ValidationError("ebe apply: dimension mismatch");
  if (u0.n_nodes != f.n_nodes || u0.batch != f.batch) throw ValidationError("solve: initial guess shape mismatch");
  const ts_solver_config c = cfg.to_c();
  const int32_t cap = cfg.residual_history_stride > 0 ? cfg.outer_max_iter / cfg.residual_history_stride + 1 : 0;
  detail::ReportBuf rb(f.batch, cap);
  VectorBatch64 u(f.n_nodes, f.batch);
  detail::finish(ts_solve(levels.handle(), f.data.data(), u0.data.data(), u.data.data(), f.n_nodes, f.batch, &c, &rb.c),
                 rb, cfg.residual_history_stride);
  return {std::move(u), rb.report(cfg.residual_history_stride)};
}

// solve_pcge (adaptive_cg.hpp:267-279): fp64 CG with the 3x3 block-Jacobi preconditioner
inline std::pair<VectorBatch64, SolveReport> solve_pcge(const EbeOperator<double>& k, const VectorBatch64& f,
                                                        const VectorBatch64& u0, double tol, int max_iter) {
  if (f.n_nodes != k.n_nodes()) throw ValidationError("ebe apply: dimension mismatch");
  if (u0.n_nodes != f.n_nodes || u0.batch != f.batch) throw ValidationError("ebe apply: dimension mismatch");
  detail::ReportBuf rb(f.batch, 0);
  VectorBatch64 u(f.n_nodes, f.batch);
  detail::finish(ts_solve_pcge(k.handle(), f.data.data(), u0.data.data(), u.data.data(), f.n_nodes, f.batch, tol,
                               max_iter, &rb.c),
                 rb, 0);
  return {std::move(u), rb.report(0)};
}

}  // namespace tetsolve
