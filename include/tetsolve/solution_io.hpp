// tetsolve/solution_io.hpp — drop-in for solution_io.hpp:12-84 (TSVEC 1).
#pragma once

#include <string>

#include "tetsolve/vector_batch.hpp"

namespace tetsolve {

inline void write_solution(const VectorBatch64& u, const std::string& path) {
  detail::check(ts_tsvec_write(path.c_str(), u.data.data(), u.n_nodes, u.batch, 0));
}
inline VectorBatch64 read_solution(const std::string& path) {
  int64_t nodes = 0;
  int32_t batch = 0;
  detail::check(ts_tsvec_info(path.c_str(), &nodes, &batch));
  VectorBatch64 u(static_cast<int32_t>(nodes), batch);
  detail::check(ts_tsvec_read(path.c_str(), u.data.data(), nodes, batch, 0));
  return u;
}

}  // namespace tetsolve
