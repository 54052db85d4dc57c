// tetsolve/solver_config.hpp — drop-in for solver_config.hpp:16-116.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "tetsolve/errors.hpp"

namespace tetsolve {

struct InnerLoopConfig {  // solver_config.hpp:16-19
  double tol = 0.1;
  int max_iter = 30;
};

struct SolverConfig {  // solver_config.hpp:21-48 (Table-2 defaults)
  double outer_tol = 1e-8;
  int outer_max_iter = 5000;
  InnerLoopConfig level0 = {0.1, 30};
  InnerLoopConfig level1 = {0.05, 300};
  InnerLoopConfig level2 = {0.025, 3000};
  int32_t batch_size = 16;
  int32_t aggregate_target = 8;
  int residual_history_stride = 1;

  ts_solver_config to_c() const {
    ts_solver_config c;
    c.outer_tol = outer_tol;
    c.outer_max_iter = outer_max_iter;
    c.level_tol[0] = level0.tol;
    c.level_tol[1] = level1.tol;
    c.level_tol[2] = level2.tol;
    c.level_max_iter[0] = level0.max_iter;
    c.level_max_iter[1] = level1.max_iter;
    c.level_max_iter[2] = level2.max_iter;
    c.batch_size = batch_size;
    c.aggregate_target = aggregate_target;
    c.residual_history_stride = residual_history_stride;
    return c;
  }
  void validate() const {
    const ts_solver_config c = to_c();
    detail::check(ts_config_validate(&c));
  }
};

struct SolveReport {  // solver_config.hpp:50-108
  bool converged = false;
  int residual_history_stride = 0;
  int outer_iterations = 0;
  long inner_iterations[3] = {0, 0, 0};
  std::vector<double> final_rel_residual;
  std::vector<std::pair<int, std::vector<double>>> residual_history;
  double time_setup_s = 0.0, time_outer_s = 0.0;
  double time_inner_s[3] = {0.0, 0.0, 0.0};
  double time_total_s = 0.0;
  int32_t batch_size = 0;
  std::string method = "amg";
  std::string inner_precision = "float32";
  double max_final_residual() const {
    double m = 0.0;
    for (double v : final_rel_residual) m = m > v ? m : v;
    return m;
  }
};

class ConvergenceError : public SolverError {  // solver_config.hpp:111-116
 public:
  ConvergenceError(const std::string& msg, SolveReport rep) : SolverError(msg), report(std::move(rep)) {}
  SolveReport report;
};

namespace detail {
struct ReportBuf {
  ts_solve_report c{};
  std::vector<double> final_, hist;
  std::vector<int32_t> hit;
  ReportBuf(int32_t batch, int32_t cap)
      : final_(batch), hist(size_t(cap > 0 ? cap : 1) * batch), hit(cap > 0 ? cap : 1) {
    c.final_rel_residual = final_.data();
    c.history = hist.data();
    c.history_iter = hit.data();
    c.history_capacity = cap;
  }
  SolveReport report(int stride) const {
    SolveReport r;
    r.converged = c.converged != 0;
    r.residual_history_stride = stride;
    r.outer_iterations = c.outer_iterations;
    for (int i = 0; i < 3; ++i) {
      r.inner_iterations[i] = static_cast<long>(c.inner_iterations[i]);
      r.time_inner_s[i] = c.time_inner_s[i];
    }
    r.final_rel_residual = final_;
    const int32_t b = static_cast<int32_t>(final_.size());
    for (int32_t i = 0; i < c.history_count; ++i)
      r.residual_history.emplace_back(hit[i], std::vector<double>(hist.begin() + size_t(i) * b,
                                                                   hist.begin() + size_t(i + 1) * b));
    r.time_setup_s = c.time_setup_s;
    r.time_outer_s = c.time_outer_s;
    r.time_total_s = c.time_total_s;
    r.batch_size = c.batch_size;
    r.method = c.method == 1 ? "pcge" : "amg";
    r.inner_precision = c.inner_precision == 64 ? "float64" : "float32";
    return r;
  }
};
inline void finish(ts_status rc, const ReportBuf& rb, int stride) {
  if (rc == TS_ERR_NO_CONVERGENCE) throw ConvergenceError(ts_last_error(), rb.report(stride));
  check(rc);
}
}  // namespace detail

}  // namespace tetsolve
