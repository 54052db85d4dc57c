// tetsolve/mesh_io.hpp — drop-in for mesh_io.hpp:13-115: TSMESH 1 text
// (byte-identical to the reference writer, atomic replace), the Dirichlet
// sidecar, and this library's TSBMESH binary mesh.
#pragma once

#include <string>
#include <vector>

#include "tetsolve/mesh.hpp"

namespace tetsolve {

inline void write_mesh(const Mesh& m, const std::string& path) {
  detail::MeshHandle h(m);
  detail::check(ts_mesh_write_tsmesh(h.h, path.c_str()));
}
inline void write_dirichlet(const Mesh& m, const std::string& path) {
  detail::MeshHandle h(m);
  detail::check(ts_mesh_write_dirichlet(h.h, path.c_str()));
}
inline Mesh read_mesh(const std::string& path) {
  ts_mesh* h = nullptr;
  detail::check(ts_mesh_read_tsmesh(path.c_str(), &h));
  return detail::take_mesh(h);
}
inline void read_dirichlet(Mesh& m, const std::string& path) {
  detail::MeshHandle h(m);
  detail::check(ts_mesh_read_dirichlet(h.h, path.c_str()));
  int32_t nn, nv, ne, nbc;
  ts_mesh_sizes(h.h, &nn, &nv, &ne, &nbc);
  std::vector<int32_t> bn(nbc);
  std::vector<int8_t> ba(nbc);
  ts_mesh_export(h.h, nullptr, nullptr, nullptr, bn.data(), ba.data());
  m.dirichlet.clear();
  for (int32_t i = 0; i < nbc; ++i) m.dirichlet.push_back({bn[i], ba[i]});
}
// TSBMESH 1: binary mesh including the Dirichlet list (no reference counterpart)
inline void write_mesh_binary(const Mesh& m, const std::string& path) {
  detail::MeshHandle h(m);
  detail::check(ts_mesh_write_tsbmesh(h.h, path.c_str()));
}
inline Mesh read_mesh_binary(const std::string& path) {
  ts_mesh* h = nullptr;
  detail::check(ts_mesh_read_tsbmesh(path.c_str(), &h));
  return detail::take_mesh(h);
}

}  // namespace tetsolve
