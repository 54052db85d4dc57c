// tetsolve/prolongation.hpp — drop-in for prolongation.hpp:10-100: nodal
// transfers with the same weights on every axis. apply / restrict_to_coarse
// run on the device in T (restriction summed in ascending fine row, the
// reference's serial scatter order: bit-identical results).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "tetsolve/mesh.hpp"
#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

struct Prolongation {  // prolongation.hpp:13-62
  enum class Kind { geometric_p1_to_p2, aggregation_l2_to_l1 };
  Kind kind = Kind::geometric_p1_to_p2;
  int32_t n_fine_nodes = 0;
  int32_t n_coarse_nodes = 0;
  std::vector<int32_t> row_ptr;
  std::vector<int32_t> cols;
  std::vector<double> weights;

  std::shared_ptr<ts_prolong> device() const {
    if (static_cast<int32_t>(row_ptr.size()) != n_fine_nodes + 1 || cols.size() != weights.size() ||
        static_cast<size_t>(row_ptr.back()) != cols.size())
      throw ValidationError("prolongation: inconsistent arrays");
    ts_prolong* h = nullptr;
    detail::check(ts_prolong_create(n_fine_nodes, n_coarse_nodes, row_ptr.data(), cols.data(), weights.data(), &h));
    return std::shared_ptr<ts_prolong>(h, ts_prolong_destroy);
  }
  // fine = P coarse
  template <typename T>
  void apply(const VectorBatch<T>& coarse, VectorBatch<T>& fine) const {
    if (coarse.n_nodes != n_coarse_nodes) throw ValidationError("prolongation apply: coarse dimension mismatch");
    if (fine.n_nodes != n_fine_nodes || fine.batch != coarse.batch) fine = VectorBatch<T>(n_fine_nodes, coarse.batch);
    if (fine.data.empty()) return;
    const auto d = device();
    detail::check(ts_prolong_apply_host(d.get(), detail::prec_of(sizeof(T)), 0, coarse.data.data(), fine.data.data(),
                                        coarse.batch));
  }
  // coarse = P^T fine
  template <typename T>
  void restrict_to_coarse(const VectorBatch<T>& fine, VectorBatch<T>& coarse) const {
    if (fine.n_nodes != n_fine_nodes) throw ValidationError("prolongation restrict: fine dimension mismatch");
    if (coarse.n_nodes != n_coarse_nodes || coarse.batch != fine.batch)
      coarse = VectorBatch<T>(n_coarse_nodes, fine.batch);
    if (coarse.data.empty()) return;
    const auto d = device();
    detail::check(ts_prolong_apply_host(d.get(), detail::prec_of(sizeof(T)), 1, fine.data.data(), coarse.data.data(),
                                        fine.batch));
  }
};

// build_geometric_prolongation (prolongation.hpp:67-98)
inline Prolongation build_geometric_prolongation(const Mesh& mesh) {
  Prolongation p;
  p.kind = Prolongation::Kind::geometric_p1_to_p2;
  p.n_fine_nodes = mesh.node_count();
  p.n_coarse_nodes = mesh.vertex_count;
  const size_t nnz = size_t(mesh.vertex_count) + 2 * size_t(mesh.node_count() - mesh.vertex_count);
  p.row_ptr.resize(size_t(p.n_fine_nodes) + 1);
  p.cols.resize(nnz);
  p.weights.resize(nnz);
  detail::MeshHandle h(mesh);
  detail::check(ts_geometric_prolongation(h.h, p.row_ptr.data(), p.cols.data(), p.weights.data()));
  return p;
}

}  // namespace tetsolve
