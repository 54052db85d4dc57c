// tetsolve/pcg.hpp — drop-in for pcg.hpp:15-126: the inner preconditioned CG
// (Algorithm 1(b)) on a batch, for an EbeOperator<T> or a BlockCsrMatrix<T>.
// The loop runs on the device (ts_inner_pcg_host): per-column scalars,
// max-over-columns termination, the stagnation and breakdown rules, fp64
// reductions. PcgWork keeps the reference's signature; the device loop owns
// its workspaces.
#pragma once

#include <cstdint>
#include <limits>
#include <type_traits>
#include <vector>

#include "tetsolve/block_csr.hpp"
#include "tetsolve/block_jacobi.hpp"
#include "tetsolve/ebe_operator.hpp"
#include "tetsolve/solver_config.hpp"
#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

struct InnerStats {  // pcg.hpp:15-18
  int iterations = 0;
  bool converged = false;
};

template <typename T>
struct PcgWork {  // pcg.hpp:22-25
  VectorBatch<T> e, z, p, q;
};

namespace detail {
// max_rel_ratio (pcg.hpp:32-42)
inline double max_rel_ratio(const std::vector<double>& num2, const std::vector<double>& den2) {
  double worst = 0.0;
  for (size_t b = 0; b < num2.size(); ++b) {
    if (den2[b] == 0.0) {
      if (num2[b] != 0.0) return std::numeric_limits<double>::infinity();
      continue;
    }
    worst = num2[b] / den2[b] > worst ? num2[b] / den2[b] : worst;
  }
  return worst;
}
template <typename Op>
struct InnerOp;
template <typename T>
struct InnerOp<EbeOperator<T>> {
  std::shared_ptr<const void> keep;
  const void* h;
  int kind = 0;
  explicit InnerOp(const EbeOperator<T>& a) : h(a.handle()) {}
};
template <typename T>
struct InnerOp<BlockCsrMatrix<T>> {
  std::shared_ptr<ts_bcsr> keep;
  const void* h;
  int kind = 1;
  explicit InnerOp(const BlockCsrMatrix<T>& a) : keep(a.device()), h(keep.get()) {}
};
}  // namespace detail

// inner_pcg (pcg.hpp:52-124)
template <typename Op, typename T>
InnerStats inner_pcg(const Op& a, const BlockJacobi<T>& m, const VectorBatch<T>& r, VectorBatch<T>& u, double tol,
                     int max_iter, PcgWork<T>& w) {
  (void)w;
  if (max_iter < 1) throw ValidationError("inner_pcg: max_iter must be >= 1");
  check_same_shape(r, u, "inner_pcg");
  const detail::InnerOp<Op> op(a);
  const auto mj = m.device();
  int32_t it = 0, conv = 0;
  detail::check(ts_inner_pcg_host(op.kind, op.h, mj.get(), r.data.data(), u.data.data(), r.n_nodes, r.batch, tol,
                                  max_iter, &it, &conv));
  InnerStats st;
  st.iterations = it;
  st.converged = conv != 0;
  return st;
}

}  // namespace tetsolve
