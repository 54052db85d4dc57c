// mesh_io.h — TSMESH / Dirichlet sidecar / TSVEC (mesh_io.hpp, solution_io.hpp)
// and the binary TSBMESH mesh; host-side, parallel (mesh_io.cc).
#pragma once
#include <array>
#include <string>
#include <vector>

#include "ts_common.h"

namespace tsg {

void validate_mesh(const Mesh& m);                            // mesh.hpp:75-113
void write_tsmesh(const Mesh& m, const std::string& path);    // mesh_io.hpp:20-36
Mesh read_tsmesh(const std::string& path);                    // mesh_io.hpp:44-96
void write_dirichlet(const Mesh& m, const std::string& path); // mesh_io.hpp:38-42
void read_dirichlet(Mesh& m, const std::string& path);        // mesh_io.hpp:98-115
void write_tsbmesh(const Mesh& m, const std::string& path);
Mesh read_tsbmesh(const std::string& path);
// solution_io.hpp:14-27 / 29-84; u = [nodes][3][batch] fp64 on the host or device
void write_tsvec(const std::string& path, const double* u, int64_t nodes, int64_t batch, bool on_device);
void tsvec_info(const std::string& path, int64_t* nodes, int64_t* batch, int64_t* data_offset);
void read_tsvec(const std::string& path, double* u, int64_t nodes, int64_t batch, bool on_device);

// Green's-sweep files: TSFAULT 1 (fault.hpp:44-84), observations (greens.hpp:20-44), TSGREENS 1
// (greens.hpp:147-222)
struct Observation {
  double p[3] = {0, 0, 0};
  int32_t axis = 0;
};
struct GreensBankData {
  int32_t rows = 0, cols = 0;
  std::vector<Observation> obs;
  std::vector<double> centers;  // [cols][3]
  std::vector<int32_t> dirs;    // 0 dip, 1 strike
  std::vector<double> radii;
  std::vector<double> values;   // row-major rows x cols
};
void write_fault_faces(const std::vector<std::array<int32_t, 3>>& faces, const std::string& path);
std::vector<std::array<int32_t, 3>> read_fault_faces(const std::string& path);
std::vector<Observation> read_observations(const std::string& path);
void write_greens_bank(const GreensBankData& g, const std::string& path);
GreensBankData read_greens_bank(const std::string& path);

}  // namespace tsg
