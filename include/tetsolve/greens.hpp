// tetsolve/greens.hpp — drop-in for greens.hpp:15-224: the Green's-function
// bank (batched slip lifting + solve + device sampling per batch) and its files.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "tetsolve/model.hpp"

namespace tetsolve {

struct ObservationComponent {  // greens.hpp:15-18
  Vec3 point{};
  int axis = 0;
};

struct GreensBank {  // greens.hpp:79-92
  struct ColumnMeta {
    Vec3 center{};
    SlipDirection direction = SlipDirection::dip;
    double radius = 0.0;
  };
  int32_t rows = 0;
  int32_t cols = 0;
  std::vector<double> values;  // row-major rows x cols
  std::vector<ObservationComponent> obs;
  std::vector<ColumnMeta> columns;
  double& at(int32_t r, int32_t c) { return values[static_cast<size_t>(r) * cols + c]; }
  double at(int32_t r, int32_t c) const { return values[static_cast<size_t>(r) * cols + c]; }
};

struct GreensReport {  // greens.hpp:95-99 (per_batch reports are not kept)
  int solver_calls = 0;
  long outer_iterations = 0;
  std::vector<SolveReport> per_batch;
};

// compute_greens_bank (greens.hpp:114-145): ceil(n / batch) solver calls
inline std::pair<GreensBank, GreensReport> compute_greens_bank(const FaultedModel& fm,
                                                               const std::vector<UnitSlip>& slips,
                                                               const std::vector<ObservationComponent>& obs,
                                                               const SolverConfig& cfg) {
  const detail::SlipArrays a(slips);
  std::vector<double> pts;
  std::vector<int32_t> axes;
  for (const auto& o : obs) {
    pts.insert(pts.end(), o.point.begin(), o.point.end());
    axes.push_back(o.axis);
  }
  GreensBank bank;
  bank.rows = static_cast<int32_t>(obs.size());
  bank.cols = static_cast<int32_t>(slips.size());
  bank.values.assign(static_cast<size_t>(bank.rows) * bank.cols, 0.0);
  bank.obs = obs;
  for (const auto& s : slips) bank.columns.push_back({s.center, s.direction, s.radius});
  const ts_solver_config c = cfg.to_c();
  GreensReport rep;
  int32_t calls = 0;
  int64_t outer = 0;
  detail::check(ts_greens_bank(fm.handle.get(), bank.cols, a.centers.data(), a.dirs.data(), a.radii.data(), bank.rows,
                               pts.data(), axes.data(), &c, bank.values.data(), &calls, &outer));
  rep.solver_calls = calls;
  rep.outer_iterations = static_cast<long>(outer);
  return {std::move(bank), std::move(rep)};
}

// read_observations (greens.hpp:20-44)
inline std::vector<ObservationComponent> read_observations(const std::string& path) {
  int32_t n = 0;
  detail::check(ts_observations_read(path.c_str(), &n, nullptr, nullptr));
  std::vector<double> p(3 * size_t(n));
  std::vector<int32_t> ax(n);
  detail::check(ts_observations_read(path.c_str(), &n, p.data(), ax.data()));
  std::vector<ObservationComponent> out(n);
  for (int32_t i = 0; i < n; ++i) out[i] = {{p[3 * i], p[3 * i + 1], p[3 * i + 2]}, ax[i]};
  return out;
}

// TSGREENS 1 banks (greens.hpp:147-222)
inline void write_greens_bank(const GreensBank& bank, const std::string& path) {
  std::vector<double> pts, centers, radii;
  std::vector<int32_t> axes, dirs;
  for (const auto& o : bank.obs) {
    pts.insert(pts.end(), o.point.begin(), o.point.end());
    axes.push_back(o.axis);
  }
  for (const auto& c : bank.columns) {
    centers.insert(centers.end(), c.center.begin(), c.center.end());
    dirs.push_back(static_cast<int32_t>(c.direction));
    radii.push_back(c.radius);
  }
  detail::check(ts_greens_bank_write(path.c_str(), bank.rows, bank.cols, pts.data(), axes.data(), centers.data(),
                                     dirs.data(), radii.data(), bank.values.data()));
}
inline GreensBank read_greens_bank(const std::string& path) {
  GreensBank b;
  detail::check(ts_greens_bank_read(path.c_str(), &b.rows, &b.cols, nullptr, nullptr, nullptr, nullptr, nullptr,
                                    nullptr));
  std::vector<double> pts(3 * size_t(b.rows)), centers(3 * size_t(b.cols)), radii(b.cols);
  std::vector<int32_t> axes(b.rows), dirs(b.cols);
  b.values.resize(size_t(b.rows) * b.cols);
  detail::check(ts_greens_bank_read(path.c_str(), &b.rows, &b.cols, pts.data(), axes.data(), centers.data(),
                                    dirs.data(), radii.data(), b.values.data()));
  for (int32_t r = 0; r < b.rows; ++r) b.obs.push_back({{pts[3 * r], pts[3 * r + 1], pts[3 * r + 2]}, axes[r]});
  for (int32_t c = 0; c < b.cols; ++c)
    b.columns.push_back({{centers[3 * c], centers[3 * c + 1], centers[3 * c + 2]},
                         dirs[c] == 0 ? SlipDirection::dip : SlipDirection::strike, radii[c]});
  return b;
}

}  // namespace tetsolve
