// levels_api.h — the single-device level set (solver.cu) for other translation units.
#pragma once
#include "ts_common.h"

namespace tsg {
ts_levels* levels_build(const Mesh& m, int32_t n_mat, const double* lam, const double* mu, const uint8_t* dof_mask,
                        const ts_solver_config& cfg);
void levels_free(ts_levels* lv);
// solve (adaptive_cg.hpp:242-263) on device buffers, serialised per level set
void levels_solve_device(ts_levels& lv, const double* f, const double* u0, double* u, int32_t B,
                         const ts_solver_config& cfg, ts_solve_report& rep, cudaStream_t s);
int32_t levels_nodes(const ts_levels& lv);
const uint8_t* levels_mask0(const ts_levels& lv);  // device [3 N] dof mask
}  // namespace tsg
