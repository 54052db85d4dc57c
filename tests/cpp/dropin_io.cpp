// The reference's file-format tests (test_mesh.cpp:120-188, test_cli.cpp's TSVEC
// round trip) written against the drop-in header: only the include changes.
// Host-only (no GPU needed). Prints one JSON line; exit code 0 = all checks held.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>

#include "tetsolve_b200/tetsolve.hpp"

using namespace tetsolve;
namespace fs = std::filesystem;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "CHECK failed line %d: %s\n", __LINE__, #c); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const fs::path dir = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "tsgpu_dropin_io";
  fs::create_directories(dir);
  int parse_throw = 0, volume_throw = 0;

  // "mesh file round-trip is bit-exact" (test_mesh.cpp:120-144)
  BoxMeshSpec spec;
  spec.extents = {1723.0, 911.0, 400.5};
  spec.divisions = {2, 3, 2};
  spec.layer_interfaces = {133.7};
  const Mesh m = generate_box_mesh(spec);
  const auto path = (dir / "roundtrip.tsmesh").string();
  const auto bc_path = (dir / "roundtrip.dirichlet").string();
  write_mesh(m, path);
  write_dirichlet(m, bc_path);
  Mesh r = read_mesh(path);
  read_dirichlet(r, bc_path);
  CHECK(r.node_count() == m.node_count());
  CHECK(r.vertex_count == m.vertex_count);
  CHECK(r.element_count() == m.element_count());
  CHECK(r.coords == m.coords);
  CHECK(r.tets10 == m.tets10);
  CHECK(r.tets4 == m.tets4);
  CHECK(r.material_id == m.material_id);
  CHECK(r.dirichlet.size() == m.dirichlet.size());
  for (size_t i = 0; i < r.dirichlet.size() && i < m.dirichlet.size(); ++i)
    CHECK(r.dirichlet[i].node == m.dirichlet[i].node && r.dirichlet[i].axis == m.dirichlet[i].axis);
  CHECK(r.edge_map == m.edge_map);

  // "truncated mesh file reports the position" (test_mesh.cpp:146-163)
  {
    std::string text;
    {
      std::ifstream is(path);
      std::string line;
      for (int i = 0; i < 10 && std::getline(is, line); ++i) text += line + "\n";
    }
    const auto tpath = (dir / "trunc.tsmesh").string();
    std::ofstream(tpath) << text;
    try {
      read_mesh(tpath);
    } catch (const ParseError& e) {
      parse_throw = std::string(e.what()).find(":11: unexpected end of file") != std::string::npos;
    }
  }
  // "negative-volume element is rejected by name" (test_mesh.cpp:165-178)
  {
    Mesh bad = m;
    std::swap(bad.tets10[3][0], bad.tets10[3][1]);
    std::swap(bad.tets4[3][0], bad.tets4[3][1]);
    const auto npath = (dir / "negvol.tsmesh").string();
    write_mesh(bad, npath);
    try {
      read_mesh(npath);
    } catch (const ParseError&) {
    } catch (const ValidationError& e) {
      volume_throw = std::string(e.what()).find("element 3") != std::string::npos;
    }
  }
  // TSVEC round trip (solution_io.hpp)
  VectorBatch64 u(m.node_count(), 3);
  for (size_t i = 0; i < u.data.size(); ++i) u.data[i] = 0.001 * double(i) - 7.0 / double(i + 1);
  const auto vpath = (dir / "u.tsvec").string();
  write_solution(u, vpath);
  const VectorBatch64 v = read_solution(vpath);
  CHECK(v.n_nodes == u.n_nodes && v.batch == u.batch && v.data == u.data);
  // binary mesh keeps the Dirichlet list
  write_mesh_binary(m, (dir / "m.tsbmesh").string());
  const Mesh b = read_mesh_binary((dir / "m.tsbmesh").string());
  CHECK(b.coords == m.coords && b.tets10 == m.tets10 && b.dirichlet.size() == m.dirichlet.size());

  CHECK(parse_throw == 1);
  CHECK(volume_throw == 1);
  std::printf("{\"failures\": %d, \"parse_throw\": %d, \"volume_throw\": %d, \"nodes\": %d}\n", failures,
              parse_throw, volume_throw, m.node_count());
  fs::remove_all(dir);
  return failures == 0 ? 0 : 1;
}
