// solver_core.h — the solve-path control loops shared by the single-device
// solver (solver.cu) and the partitioned one (dist_solver.cu): inner PCG
// (pcg.hpp:52-124) and the fp64 flexible outer CG (adaptive_cg.hpp:126-233).
// Operators and preconditioners are callables; distributed runs set
// Workspace::comm / ::owned so the same loops reduce across ranks.
#pragma once
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "blas.h"
#include "ebe.h"

namespace tsg {
namespace core {

using clk = std::chrono::steady_clock;
inline double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

inline const PcgStatus& read_status(Workspace& ws, cudaStream_t s) {
  TS_CUDA(cudaMemcpyAsync(ws.host_status, ws.status.get(), sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
  TS_CUDA(cudaStreamSynchronize(s));
  return *ws.host_status;
}

struct InnerStats {
  int iterations = 0;
  bool converged = false;
};

// inner_pcg (pcg.hpp:52-124). A(x, y, init): y = A x on the stream; with
// fuse_init the direction pass writes A's starting value (the masked identity
// of p, op_mask = the operator's dof mask) and A is called with init = false.
template <typename T, typename Op>
InnerStats inner_pcg(Op&& A, const T* inv, const T* r, T* u, int32_t n, int32_t B, double tol, int max_iter, T* e,
                     T* p, T* q, ColScalars& cs, Workspace& ws, cudaStream_t s, bool fuse_init = false,
                     const uint8_t* op_mask = nullptr,
                     const std::function<int(const T*, T*)>* product_with_dots = nullptr) {
  if (max_iter < 1) validation("inner_pcg: max_iter must be >= 1");
  A(u, e, true);
  pcg_init<T>(inv, r, e, n, B, cs, ws, s);
  InnerStats st;
  const double tol2 = tol * tol;
  double ratio = read_status(ws, s).ratio;
  if (std::isnan(ratio)) fail(TS_ERR_NONFINITE, "inner_pcg: non-finite initial residual");
  // u += alpha p of the last completed iteration, folded into the next direction pass
  // (which reads the old p anyway) or applied once after the loop
  bool pending = false;
  while (ratio > tol2 && st.iterations < max_iter) {
    const bool first = st.iterations == 0;
    pcg_rho(B, first, cs, ws, s);
    pcg_direction<T>(inv, e, p, n, B, first, cs, s, fuse_init ? q : nullptr, op_mask, pending ? u : nullptr);
    pending = false;
    // q = A p; gamma's partials from the product itself when it can (1: all three dots, assembled
    // levels; 2: (p,Ap) alone, element-wise on the EBE level), else a separate pass
    const int fused = product_with_dots ? (*product_with_dots)(p, q) : 0;
    if (fused) {
      pcg_gamma_final<T>(B, cs, ws, s, fused == 2);
    } else {
      A(p, q, !fuse_init);
      pcg_gamma<T>(p, q, n, B, cs, ws, s);
    }
    pcg_update<T>(inv, e, q, n, B, cs, ws, s);
    const PcgStatus* psp = &read_status(ws, s);
    if (psp->need_full) {  // (p,Ap) <= 0 in some column: decide it with the full dots (pcg.hpp:83-110)
      pcg_gamma<T>(p, q, n, B, cs, ws, s);
      pcg_update<T>(inv, e, q, n, B, cs, ws, s);
      psp = &read_status(ws, s);
    }
    const PcgStatus& ps = *psp;
    if (ps.breakdown_col >= 0)
      fail(TS_ERR_BREAKDOWN, "inner_pcg: breakdown (p,Ap) <= 0 at iteration " + std::to_string(st.iterations + 1) +
                                 ", column " + std::to_string(ps.breakdown_col));
    if (ps.stagnated) break;  // the reference leaves u and e as they were (pcg.hpp:99-104)
    pending = true;
    ++st.iterations;
    ratio = ps.ratio;
    if (std::isnan(ratio))
      fail(TS_ERR_NONFINITE, "inner_pcg: non-finite residual at iteration " + std::to_string(st.iterations));
  }
  if (pending) pcg_apply_pending<T>(u, p, n, B, cs, s);
  st.converged = ratio <= tol2;
  return st;
}

inline void report_reset(ts_solve_report& rep, int method, int prec) {
  rep.converged = 0;
  rep.outer_iterations = 0;
  for (int i = 0; i < 3; ++i) {
    rep.inner_iterations[i] = 0;
    rep.time_inner_s[i] = 0.0;
  }
  rep.time_setup_s = rep.time_outer_s = rep.time_total_s = 0.0;
  rep.history_count = 0;
  rep.method = method;
  rep.inner_precision = prec;
}

// run_outer_cg (adaptive_cg.hpp:126-233); vectors r,q,z,p,scratch of `lv.v`.
// K(x, y): y = K x (fp64 outer operator) on n nodes; vectors r,q,z,p of `v`.
template <typename Vecs, typename KOp, typename Precond>
void run_outer_cg(KOp&& K, int32_t n, const double* f, double* u, int32_t B, double tol, int max_iter, int stride,
                  Precond&& precond, Vecs& v, ColScalars& cs, Workspace& ws, ts_solve_report& rep,
                  cudaStream_t s) {
  const auto t_start = clk::now();
  std::vector<double> fn2(B), rn2(B);
  dot2<double>(f, f, nullptr, nullptr, 3 * int64_t(n), B, cs[ColScalars::FN2], ws, s);
  TS_CUDA(cudaMemcpyAsync(fn2.data(), cs[ColScalars::FN2], B * sizeof(double), cudaMemcpyDeviceToHost, s));
  auto true_residual = [&]() -> double {
    K(u, v.r.get());
    cg_true_residual(f, v.r.get(), n, B, cs, ws, s);
    return read_status(ws, s).ratio;
  };
  auto finalize = [&]() {
    TS_CUDA(cudaMemcpyAsync(rn2.data(), cs[ColScalars::RN2], B * sizeof(double), cudaMemcpyDeviceToHost, s));
    TS_CUDA(cudaStreamSynchronize(s));
    rep.batch_size = B;
    if (rep.final_rel_residual)
      for (int b = 0; b < B; ++b)
        rep.final_rel_residual[b] = fn2[b] > 0.0 ? std::sqrt(rn2[b] / fn2[b])
                                                 : (rn2[b] > 0.0 ? std::numeric_limits<double>::infinity() : 0.0);
    rep.time_total_s = secs(t_start, clk::now());
    rep.time_outer_s = rep.time_total_s - rep.time_inner_s[0] - rep.time_inner_s[1] - rep.time_inner_s[2];
  };
  double ratio = true_residual();
  const double tol2 = tol * tol;
  rep.batch_size = B;
  int it = 0;
  bool r_is_true = true, first = true;
  while (true) {
    if (std::isnan(ratio)) fail(TS_ERR_NONFINITE, "solve: non-finite residual");
    if (ratio <= tol2) {
      if (r_is_true) break;
      ratio = true_residual();
      r_is_true = true;
      if (ratio <= tol2) break;
    }
    if (it >= max_iter) {
      if (!r_is_true) ratio = true_residual();
      rep.outer_iterations = it;
      rep.converged = 0;
      finalize();
      char buf[64];
      std::snprintf(buf, sizeof buf, "%f", std::sqrt(ratio));
      fail(TS_ERR_NO_CONVERGENCE, "solve: outer loop did not converge within " + std::to_string(max_iter) +
                                      " iterations (max residual " + buf + ")");
    }
    precond(v.r.get(), v.z.get());
    cg_direction(v.z.get(), v.q.get(), v.p.get(), n, B, first, cs, ws, s);
    first = false;
    K(v.p.get(), v.q.get());
    cg_alpha(v.z.get(), v.r.get(), v.p.get(), v.q.get(), n, B, cs, ws, s);
    cg_update(v.r.get(), u, v.p.get(), v.q.get(), n, B, cs, ws, s);
    const PcgStatus& ps = read_status(ws, s);
    if (ps.breakdown_col >= 0)
      fail(TS_ERR_BREAKDOWN, "solve: breakdown (p,Kp) <= 0 at outer iteration " + std::to_string(it + 1) +
                                 ", column " + std::to_string(ps.breakdown_col));
    ratio = ps.ratio;
    r_is_true = false;
    ++it;
    if (stride > 0 && it % stride == 0 && rep.history_count < rep.history_capacity) {
      TS_CUDA(cudaMemcpyAsync(rn2.data(), cs[ColScalars::RN2], B * sizeof(double), cudaMemcpyDeviceToHost, s));
      TS_CUDA(cudaStreamSynchronize(s));
      const int32_t row = rep.history_count++;
      if (rep.history_iter) rep.history_iter[row] = it;
      if (rep.history)
        for (int b = 0; b < B; ++b)
          rep.history[size_t(row) * B + b] = fn2[b] > 0.0 ? std::sqrt(rn2[b] / fn2[b]) : 0.0;
    }
  }
  rep.outer_iterations = it;
  rep.converged = 1;
  finalize();
}


}  // namespace core
}  // namespace tsg
