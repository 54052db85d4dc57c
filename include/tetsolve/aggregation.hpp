// tetsolve/aggregation.hpp — drop-in for aggregation.hpp:13-187: the greedy
// aggregation of the first-order operator, the Galerkin level 2 and the
// coarse mask. The library's setup code (the reference's sequential,
// order-exact algorithm, csrc/setup.cpp) computes them; build_solver_levels
// runs the same code.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "tetsolve/block_csr.hpp"
#include "tetsolve/prolongation.hpp"

namespace tetsolve {

struct Aggregation {  // aggregation.hpp:13-17
  std::vector<int32_t> agg_of_node;
  int32_t n_aggregates = 0;
  std::vector<int32_t> seeds;  // seed node of each aggregate, in creation order
};

// aggregate_p1 (aggregation.hpp:23-89)
inline Aggregation aggregate_p1(const BlockCsrMatrix<double>& a, int32_t target_size) {
  Aggregation agg;
  agg.agg_of_node.resize(a.n_block_rows);
  std::vector<int32_t> seeds(a.n_block_rows);
  detail::check(ts_aggregate_p1(a.n_block_rows, a.row_ptr.data(), a.col_idx.data(), target_size,
                                agg.agg_of_node.data(), &agg.n_aggregates, seeds.data()));
  agg.seeds.assign(seeds.begin(), seeds.begin() + agg.n_aggregates);
  return agg;
}

// build_level2 (aggregation.hpp:95-170): aggregation prolongation P2 and A2 = P2^T K1 P2
inline std::pair<Prolongation, BlockCsrMatrix<double>> build_level2(const BlockCsrMatrix<double>& k1,
                                                                    const Aggregation& agg,
                                                                    const std::vector<uint8_t>& fine_mask = {}) {
  const int32_t nf = k1.n_block_rows;
  if (static_cast<int32_t>(agg.agg_of_node.size()) != nf)
    throw ValidationError("build_level2: aggregation size mismatch");
  const uint8_t* mk = fine_mask.empty() ? nullptr : fine_mask.data();
  int64_t nnzb2 = 0;
  detail::check(ts_build_level2(nf, k1.row_ptr.data(), k1.col_idx.data(), k1.blocks.empty() ? nullptr : k1.blocks[0].data(),
                                agg.agg_of_node.data(), agg.n_aggregates, mk, &nnzb2, nullptr, nullptr, nullptr));
  BlockCsrMatrix<double> a2;
  a2.n_block_rows = agg.n_aggregates;
  a2.row_ptr.resize(size_t(agg.n_aggregates) + 1);
  a2.col_idx.resize(nnzb2);
  a2.blocks.resize(nnzb2);
  detail::check(ts_build_level2(nf, k1.row_ptr.data(), k1.col_idx.data(), k1.blocks.empty() ? nullptr : k1.blocks[0].data(),
                                agg.agg_of_node.data(), agg.n_aggregates, mk, &nnzb2, a2.row_ptr.data(),
                                a2.col_idx.data(), a2.blocks.empty() ? nullptr : a2.blocks[0].data()));
  Prolongation p;
  p.kind = Prolongation::Kind::aggregation_l2_to_l1;
  p.n_fine_nodes = nf;
  p.n_coarse_nodes = agg.n_aggregates;
  p.row_ptr.resize(size_t(nf) + 1);
  for (int32_t i = 0; i <= nf; ++i) p.row_ptr[i] = i;
  p.cols = agg.agg_of_node;
  p.weights.assign(nf, 1.0);
  return {std::move(p), std::move(a2)};
}

// coarse_mask (aggregation.hpp:174-185): a coarse dof is constrained when every fine node of
// its aggregate is constrained on that axis (flag bookkeeping)
inline std::vector<uint8_t> coarse_mask(const Aggregation& agg, const std::vector<uint8_t>& fine_mask) {
  std::vector<uint8_t> out(static_cast<size_t>(3) * agg.n_aggregates, fine_mask.empty() ? 0 : 1);
  if (fine_mask.empty()) return out;
  for (size_t node = 0; node < agg.agg_of_node.size(); ++node)
    for (int i = 0; i < 3; ++i)
      if (!fine_mask[3 * node + i]) out[3 * static_cast<size_t>(agg.agg_of_node[node]) + i] = 0;
  return out;
}

}  // namespace tetsolve
