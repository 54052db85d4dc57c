// tetsolve/material.hpp — drop-in for material.hpp:14-34.
#pragma once

#include <utility>
#include <vector>

#include "tetsolve/errors.hpp"

namespace tetsolve {

struct Material {  // material.hpp:14-20
  double vp = 0.0, vs = 0.0, rho = 0.0, lambda = 0.0, mu = 0.0;
};

// material_from_wavespeeds (material.hpp:22-34): mu = rho vs^2, lambda = rho (vp^2 - 2 vs^2)
inline Material material_from_wavespeeds(double vp, double vs, double rho) {
  Material m;
  m.vp = vp;
  m.vs = vs;
  m.rho = rho;
  detail::check(ts_material_from_wavespeeds(vp, vs, rho, &m.lambda, &m.mu));
  return m;
}

namespace detail {
inline std::pair<std::vector<double>, std::vector<double>> lame(const std::vector<Material>& mats) {
  std::vector<double> l(mats.size()), m(mats.size());
  for (size_t i = 0; i < mats.size(); ++i) {
    l[i] = mats[i].lambda;
    m[i] = mats[i].mu;
  }
  return {l, m};
}
}  // namespace detail

}  // namespace tetsolve
