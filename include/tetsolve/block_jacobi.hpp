// tetsolve/block_jacobi.hpp — drop-in for block_jacobi.hpp:12-87: inverse
// 3x3 node blocks; apply and the extraction from a block-CSR matrix run on
// the device (fp64 math rounded to T; singular blocks -> ValidationError
// naming the node, as invert_node_block).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "tetsolve/block_csr.hpp"
#include "tetsolve/geometry.hpp"
#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

template <typename T>
struct BlockJacobi {  // block_jacobi.hpp:15-39
  std::vector<std::array<T, 9>> inv_blocks;
  int32_t n_nodes() const { return static_cast<int32_t>(inv_blocks.size()); }
  std::shared_ptr<ts_bj> device() const {
    ts_bj* h = nullptr;
    detail::check(ts_bj_create(n_nodes(), inv_blocks.empty() ? nullptr : inv_blocks[0].data(),
                               detail::prec_of(sizeof(T)), &h));
    return std::shared_ptr<ts_bj>(h, ts_bj_destroy);
  }
  // z = M^-1 r (block_jacobi.hpp:22-38)
  void apply(const VectorBatch<T>& r, VectorBatch<T>& z) const {
    if (r.n_nodes != n_nodes()) throw ValidationError("block jacobi apply: dimension mismatch");
    if (z.n_nodes != r.n_nodes || z.batch != r.batch) z = VectorBatch<T>(r.n_nodes, r.batch);
    if (r.data.empty()) return;
    const auto d = device();
    detail::check(ts_bj_apply_host(d.get(), r.data.data(), z.data.data(), r.batch));
  }
};

// extract_block_jacobi(BlockCsrMatrix) (block_jacobi.hpp:72-85)
template <typename T>
inline BlockJacobi<T> extract_block_jacobi(const BlockCsrMatrix<T>& a) {
  BlockJacobi<T> m;
  m.inv_blocks.resize(a.n_block_rows);
  if (a.n_block_rows == 0) return m;
  const auto d = a.device();
  detail::check(ts_bcsr_block_jacobi_host(d.get(), m.inv_blocks.empty() ? nullptr : m.inv_blocks[0].data()));
  return m;
}

}  // namespace tetsolve
