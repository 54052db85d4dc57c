// dist_api.h — entry points of the partitioned solve (dist_solver.cu) for the C ABI.
#pragma once
#include "comm.h"
#include "ts_common.h"

namespace tsg {
ts_dist_levels* dist_levels_create(const Mesh& m, int32_t n_mat, const double* lam, const double* mu,
                                   const uint8_t* dof_mask, const int32_t* part, const ts_solver_config& cfg,
                                   Comm* comm);
void dist_levels_destroy(ts_dist_levels* L);
void dist_levels_sizes(const ts_dist_levels& L, int32_t* n0, int32_t* n1, int32_t* n2);
const std::vector<int32_t>& dist_local_nodes(const ts_dist_levels& L);
void dist_levels_info(const ts_dist_levels& L, int32_t* n_elements, int64_t* halo_rows0, int32_t* n_nbr,
                      double* setup_s);
void dist_solve_device(ts_dist_levels& L, const double* f, const double* u0, double* u, int32_t B,
                       const ts_solver_config& cfg, ts_solve_report& rep, cudaStream_t s);
void dist_solve_host(ts_dist_levels& L, const double* f, const double* u0, double* u, int32_t B,
                     const ts_solver_config& cfg, ts_solve_report& rep);
void dist_ebe_apply(ts_dist_levels& L, int which, const void* u, void* f, int32_t B, cudaStream_t s);
ts_dist_ebe* dist_ebe_create(const Mesh& m, int order, int32_t n_mat, const double* lam, const double* mu,
                             const uint8_t* dof_mask, const int32_t* part, int prec, Comm* comm);
void dist_ebe_destroy(ts_dist_ebe* D);
void dist_ebe_info(const ts_dist_ebe& D, int32_t* n_local, int32_t* n_elems, int64_t* halo_rows, int32_t* n_nbr);
const std::vector<int32_t>& dist_ebe_local_nodes(const ts_dist_ebe& D);
void dist_ebe_apply_op(ts_dist_ebe& D, const void* u, void* f, int32_t B, cudaStream_t s);
ts_ebe* dist_ebe_local(ts_dist_ebe& D);
Comm* dist_levels_comm(const ts_dist_levels& L);
const uint8_t* dist_levels_mask0(const ts_dist_levels& L);  // device [3 n_local] dof mask
Comm* dist_ebe_comm(const ts_dist_ebe& D);
}  // namespace tsg
