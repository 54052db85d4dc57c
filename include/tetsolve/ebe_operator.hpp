// tetsolve/ebe_operator.hpp — drop-in for ebe_operator.hpp:20-315: the
// matrix-free multi-case operator f = mask_id(u) + sum_e Q_e K_e Q_e^T u,
// its element matrices, the assembled block-CSR image and the block-Jacobi
// extraction. The operator lives on the GPU (ts_ebe_*). Like the reference
// (SPEC determinism, ebe_operator.hpp:25-28) its products are deterministic:
// an operator built here sweeps its elements by color (ts_ebe_set_deterministic),
// so results are bitwise reproducible and each column's bits do not depend on
// the batch width, whatever `workers` says (accepted, unused).
// set_deterministic(false) selects the faster atomic face-pair sweep, which
// agrees to rounding.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "tetsolve/block_csr.hpp"
#include "tetsolve/block_jacobi.hpp"
#include "tetsolve/material.hpp"
#include "tetsolve/mesh.hpp"
#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

template <typename T>
class EbeOperator {  // ebe_operator.hpp:29-226
 public:
  EbeOperator() = default;
  // EbeOperator(mesh, order, materials, dof_mask, workers) (ebe_operator.hpp:35-65)
  EbeOperator(const Mesh& mesh, int order, const std::vector<Material>& materials, std::vector<uint8_t> dof_mask,
              int workers = 1)
      : order_(order), mask_(std::move(dof_mask)) {
    (void)workers;
    detail::MeshHandle mh(mesh);
    auto [l, m] = detail::lame(materials);
    ts_ebe* h = nullptr;
    detail::check(ts_ebe_create(mh.h, order, static_cast<int32_t>(l.size()), l.data(), m.data(),
                                mask_.empty() ? nullptr : mask_.data(), detail::prec_of(sizeof(T)), &h));
    op_ = std::shared_ptr<ts_ebe>(h, ts_ebe_destroy);
    detail::check(ts_ebe_set_deterministic(h, 1));
    int32_t nn = 0, ne = 0;
    detail::check(ts_ebe_info(h, &nn, &ne, nullptr, nullptr));
    n_nodes_ = nn;
    n_elems_ = ne;
    conn_ = std::make_shared<std::vector<int32_t>>(static_cast<size_t>(nodes_per_element()) * ne);
    for (int32_t e = 0; e < ne; ++e)
      for (int a = 0; a < nodes_per_element(); ++a) (*conn_)[static_cast<size_t>(nodes_per_element()) * e + a] = mesh.tets10[e][a];
  }
  // view of an operator owned elsewhere (the operators inside a SolverLevels)
  EbeOperator(std::shared_ptr<ts_ebe> op, int32_t n_nodes, int32_t n_elems, int order,
              std::shared_ptr<std::vector<int32_t>> conn, std::vector<uint8_t> mask)
      : op_(std::move(op)), order_(order), n_nodes_(n_nodes), n_elems_(n_elems), mask_(std::move(mask)),
        conn_(std::move(conn)) {}

  int32_t n_nodes() const { return n_nodes_; }
  int32_t n_elements() const { return n_elems_; }
  int order() const { return order_; }
  int nodes_per_element() const { return order_ == 1 ? 4 : 10; }
  const std::vector<uint8_t>& mask() const { return mask_; }
  int32_t element_node(int32_t e, int a) const { return (*conn_)[static_cast<size_t>(nodes_per_element()) * e + a]; }

  // element_matrix (ebe_operator.hpp:78-87): fp64 K_e of the operator's T-rounded element data
  void element_matrix(int32_t e, double* k) const { detail::check(ts_ebe_element_matrix(op_.get(), e, k)); }

  // f = A u for every batch column (ebe_operator.hpp:90-134)
  void apply(const VectorBatch<T>& u, VectorBatch<T>& f) const {
    if (u.n_nodes != n_nodes_) throw ValidationError("ebe apply: dimension mismatch");
    if (f.n_nodes != u.n_nodes || f.batch != u.batch) f = VectorBatch<T>(u.n_nodes, u.batch);
    if (u.data.empty()) return;
    detail::check(ts_ebe_apply_host(op_.get(), u.data.data(), f.data.data(), u.batch));
  }
  // device-pointer entry for callers that keep vectors in HBM
  void apply_device(const T* u, T* f, int32_t batch, void* stream = nullptr) const {
    detail::check(ts_ebe_apply(op_.get(), u, f, batch, stream));
  }
  const ts_ebe* handle() const { return op_.get(); }
  // deterministic colored sweep (default) or the atomic face-pair sweep
  void set_deterministic(bool on) { detail::check(ts_ebe_set_deterministic(op_.get(), on ? 1 : 0)); }

 private:
  std::shared_ptr<ts_ebe> op_;
  int order_ = 2;
  int32_t n_nodes_ = 0, n_elems_ = 0;
  std::vector<uint8_t> mask_;
  std::shared_ptr<std::vector<int32_t>> conn_ = std::make_shared<std::vector<int32_t>>();
};

// assemble_bcsr (ebe_operator.hpp:230-284): identity rows at constrained dofs,
// constrained columns dropped; assembled on the device in element order
template <typename T>
inline BlockCsrMatrix<T> assemble_bcsr(const EbeOperator<T>& op) {
  BlockCsrMatrix<T> a;
  a.n_block_rows = op.n_nodes();
  int64_t nnzb = 0;
  detail::check(ts_ebe_assemble_bcsr(op.handle(), &nnzb, nullptr, nullptr, nullptr));
  a.row_ptr.resize(static_cast<size_t>(op.n_nodes()) + 1);
  a.col_idx.resize(nnzb);
  a.blocks.resize(nnzb);
  detail::check(ts_ebe_assemble_bcsr(op.handle(), &nnzb, a.row_ptr.data(), a.col_idx.data(),
                                     a.blocks.empty() ? nullptr : a.blocks[0].data()));
  return a;
}

// extract_block_jacobi(EbeOperator) (ebe_operator.hpp:288-313), computed on the GPU
template <typename T>
inline BlockJacobi<T> extract_block_jacobi(const EbeOperator<T>& op) {
  BlockJacobi<T> m;
  m.inv_blocks.resize(op.n_nodes());
  if (op.n_nodes() == 0) return m;
  detail::check(ts_ebe_block_jacobi_host(op.handle(), m.inv_blocks[0].data()));
  return m;
}

}  // namespace tetsolve
