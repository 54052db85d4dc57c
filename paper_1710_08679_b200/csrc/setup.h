// setup.h — host-side hierarchy construction (see setup.cpp).
#pragma once
#include <vector>

#include "ts_common.h"

namespace tsg {

// 3x3-block CSR with fp64 values (BlockCsrMatrix<double>, block_csr.hpp:16-70)
struct BcsrD {
  int32_t n = 0;
  std::vector<int32_t> row_ptr;
  HostVec<int32_t> col_idx;
  HostVec<double> blocks;  // [nnzb][9]
};

struct Aggregation {  // aggregation.hpp:13-17
  std::vector<int32_t> agg_of_node;
  int32_t n_aggregates = 0;
  std::vector<int32_t> seeds;  // seed node of each aggregate, creation order
};

// K1 (fp64, the reference's assembly); blocks32 (optional) receives the fp32
// operator's float-rounded image on the same pattern
BcsrD assemble_tet4(const Mesh& m, const std::vector<double>& lam_e, const std::vector<double>& mu_e,
                    const std::vector<uint8_t>& mask1, HostVec<float>* blocks32 = nullptr);
Aggregation aggregate_p1(const BcsrD& a, int32_t target);
BcsrD build_level2(const BcsrD& k1, const Aggregation& agg, const std::vector<uint8_t>& fine_mask);
std::vector<uint8_t> coarse_mask(const Aggregation& agg, const std::vector<uint8_t>& fine_mask);
std::vector<float> bcsr_block_jacobi_f32(const BcsrD& a);

// Level 2 of build_solver_levels (adaptive_cg.hpp:53-65) from the GLOBAL mesh: K1 assembly,
// the sequential aggregation, the Galerkin product, its block Jacobi and coarse mask, as the
// fp32 arrays the device level uses (host-only; the partitioned setup builds it on one rank)
struct Level2Host {
  int32_t n2 = 0;
  std::vector<int32_t> agg_of_node, seeds, row_ptr, col_idx;
  std::vector<float> blocks, m2;
  std::vector<uint8_t> mask2;
};
Level2Host build_level2_host(const Mesh& m, const std::vector<double>& lam_e, const std::vector<double>& mu_e,
                             const std::vector<uint8_t>& mask1, int32_t aggregate_target);

}  // namespace tsg
