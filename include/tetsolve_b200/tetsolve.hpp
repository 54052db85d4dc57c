// tetsolve_b200/tetsolve.hpp — drop-in C++ mirror of the reference solve-path
// interface (/root/reference/proj/include/tetsolve, namespace tetsolve), backed
// by libtsgpu.so (include/tsgpu.h). A reference user replaces
//   #include "tetsolve/adaptive_cg.hpp" / "tetsolve/model.hpp"
// with
//   #include "tetsolve_b200/tetsolve.hpp"
// and links -ltsgpu. Types, signatures, ownership (value types, host
// VectorBatch in/out) and exceptions follow the reference; each symbol cites
// the reference declaration it replaces. All arithmetic runs on the GPU.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../tsgpu.h"

namespace tetsolve {

// ------------------------------------------------------------ errors.hpp:9-31
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ValidationError : public Error {
 public:
  explicit ValidationError(const std::string& m) : Error(m) {}
};
class ParseError : public ValidationError {  // errors.hpp:21-25: "file:line: msg"
 public:
  explicit ParseError(const std::string& msg) : ValidationError(msg) {}
  ParseError(const std::string& file, long line, const std::string& msg)
      : ValidationError(file + ":" + std::to_string(line) + ": " + msg) {}
};

class SolverError : public Error {
 public:
  explicit SolverError(const std::string& m) : Error(m) {}
};
class DeviceError : public Error {  // no reference counterpart: CUDA failure / no device
 public:
  explicit DeviceError(const std::string& m) : Error(m) {}
};

// ---------------------------------------------------------- geometry / material
using Vec3 = std::array<double, 3>;  // geometry.hpp:8

struct Material {  // material.hpp:14-20
  double vp = 0.0, vs = 0.0, rho = 0.0, lambda = 0.0, mu = 0.0;
};

// ------------------------------------------------------- solver_config.hpp:16-116
struct InnerLoopConfig {
  double tol = 0.1;
  int max_iter = 30;
};

struct SolverConfig {
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
  void validate() const;
};

struct SolveReport {
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

class ConvergenceError : public SolverError {
 public:
  ConvergenceError(const std::string& msg, SolveReport rep) : SolverError(msg), report(std::move(rep)) {}
  SolveReport report;
};

namespace detail {
inline void check(ts_status rc) {
  if (rc == TS_OK) return;
  const std::string msg = ts_last_error();
  switch (rc) {
    case TS_ERR_PARSE: throw ParseError(msg);
    case TS_ERR_VALIDATION: throw ValidationError(msg);
    case TS_ERR_BREAKDOWN:
    case TS_ERR_NONFINITE: throw SolverError(msg);
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

inline void SolverConfig::validate() const {
  const ts_solver_config c = to_c();
  detail::check(ts_config_validate(&c));
}

inline Material material_from_wavespeeds(double vp, double vs, double rho) {  // material.hpp:22-34
  Material m;
  m.vp = vp;
  m.vs = vs;
  m.rho = rho;
  detail::check(ts_material_from_wavespeeds(vp, vs, rho, &m.lambda, &m.mu));
  return m;
}

// ------------------------------------------------------------- mesh.hpp:19-156
struct DirichletBc {
  int32_t node = 0;
  int8_t axis = 0;
};

struct Mesh {  // vertices first; tets10 = 4 vertices + 6 edge nodes
  std::vector<Vec3> coords;
  std::vector<std::array<int32_t, 10>> tets10;
  std::vector<std::array<int32_t, 4>> tets4;
  std::vector<int32_t> material_id;
  std::map<std::pair<int32_t, int32_t>, int32_t> edge_map;
  int32_t vertex_count = 0;
  std::vector<DirichletBc> dirichlet;
  int32_t node_count() const { return static_cast<int32_t>(coords.size()); }
  int32_t element_count() const { return static_cast<int32_t>(tets10.size()); }
};

inline std::vector<uint8_t> dirichlet_mask(const Mesh& m) {  // mesh.hpp:150-154
  std::vector<uint8_t> mask(3 * static_cast<size_t>(m.node_count()), 0);
  for (const auto& bc : m.dirichlet) mask[3 * static_cast<size_t>(bc.node) + bc.axis] = 1;
  return mask;
}

enum class FixedBoundary { none, bottom_and_sides, all_clamped };  // box_mesh.hpp:13-17

struct BoxMeshSpec {  // box_mesh.hpp:23-28
  Vec3 extents = {1.0, 1.0, 1.0};
  std::array<int32_t, 3> divisions = {1, 1, 1};
  std::vector<double> layer_interfaces;
  FixedBoundary fixed_boundary = FixedBoundary::bottom_and_sides;
};

namespace detail {
struct MeshHandle {
  ts_mesh* h = nullptr;
  explicit MeshHandle(const Mesh& m) {
    std::vector<double> c(3 * m.coords.size());
    for (size_t i = 0; i < m.coords.size(); ++i)
      for (int k = 0; k < 3; ++k) c[3 * i + k] = m.coords[i][k];
    std::vector<int32_t> t(10 * m.tets10.size());
    for (size_t e = 0; e < m.tets10.size(); ++e)
      for (int a = 0; a < 10; ++a) t[10 * e + a] = m.tets10[e][a];
    std::vector<int32_t> bn(m.dirichlet.size());
    std::vector<int8_t> ba(m.dirichlet.size());
    for (size_t i = 0; i < m.dirichlet.size(); ++i) {
      bn[i] = m.dirichlet[i].node;
      ba[i] = m.dirichlet[i].axis;
    }
    check(ts_mesh_from_arrays(m.node_count(), m.vertex_count, c.data(), m.element_count(), t.data(),
                              m.material_id.data(), static_cast<int32_t>(bn.size()), bn.data(), ba.data(), &h));
  }
  ~MeshHandle() { ts_mesh_destroy(h); }
  MeshHandle(const MeshHandle&) = delete;
  MeshHandle& operator=(const MeshHandle&) = delete;
};

inline std::pair<std::vector<double>, std::vector<double>> lame(const std::vector<Material>& mats) {
  std::vector<double> l(mats.size()), m(mats.size());
  for (size_t i = 0; i < mats.size(); ++i) {
    l[i] = mats[i].lambda;
    m[i] = mats[i].mu;
  }
  return {l, m};
}
}  // namespace detail

namespace detail {
// copy a library mesh handle into the reference's Mesh (edge_map rebuilt as rebuild_edge_map, mesh.hpp:61-71)
inline Mesh take_mesh(ts_mesh* h) {
  int32_t nn, nv, ne, nbc;
  ts_mesh_sizes(h, &nn, &nv, &ne, &nbc);
  std::vector<double> c(3 * size_t(nn));
  std::vector<int32_t> t(10 * size_t(ne)), mat(ne), bn(nbc);
  std::vector<int8_t> ba(nbc);
  ts_mesh_export(h, c.data(), t.data(), mat.data(), bn.data(), ba.data());
  ts_mesh_destroy(h);
  Mesh m;
  m.vertex_count = nv;
  m.coords.resize(nn);
  for (int32_t i = 0; i < nn; ++i) m.coords[i] = {c[3 * size_t(i)], c[3 * size_t(i) + 1], c[3 * size_t(i) + 2]};
  m.tets10.resize(ne);
  m.tets4.resize(ne);
  static constexpr int ee[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  for (int32_t e = 0; e < ne; ++e) {
    for (int a = 0; a < 10; ++a) m.tets10[e][a] = t[10 * size_t(e) + a];
    for (int a = 0; a < 4; ++a) m.tets4[e][a] = t[10 * size_t(e) + a];
    for (int q = 0; q < 6; ++q) {
      int32_t a = m.tets10[e][ee[q][0]], b = m.tets10[e][ee[q][1]];
      if (a > b) std::swap(a, b);
      m.edge_map[{a, b}] = m.tets10[e][4 + q];
    }
  }
  m.material_id = std::move(mat);
  for (int32_t i = 0; i < nbc; ++i) m.dirichlet.push_back({bn[i], ba[i]});
  return m;
}
}  // namespace detail

// generate_box_mesh (box_mesh.hpp:55-157): identical node numbering
inline Mesh generate_box_mesh(const BoxMeshSpec& spec) {
  ts_mesh* h = nullptr;
  detail::check(ts_box_mesh(spec.extents.data(), spec.divisions.data(),
                            static_cast<int32_t>(spec.layer_interfaces.size()), spec.layer_interfaces.data(),
                            static_cast<int32_t>(spec.fixed_boundary), &h));
  return detail::take_mesh(h);
}

// ------------------------------------------------------------ mesh_io.hpp:13-115
// TSMESH 1 text (byte-identical to the reference writer, atomic replace) and the
// Dirichlet sidecar; read_mesh throws ParseError / ValidationError like the reference.
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

// ------------------------------------------------------- vector_batch.hpp:15-34
template <typename T>
struct VectorBatch {
  int32_t n_nodes = 0;
  int32_t batch = 0;
  std::vector<T> data;
  VectorBatch() = default;
  VectorBatch(int32_t nodes, int32_t b) : n_nodes(nodes), batch(b) {
    data.assign(static_cast<size_t>(3) * nodes * b, T(0));
  }
  int64_t n_dofs() const { return static_cast<int64_t>(3) * n_nodes; }
  T& at(int64_t dof, int32_t b) { return data[dof * batch + b]; }
  T at(int64_t dof, int32_t b) const { return data[dof * batch + b]; }
  void set_zero() { std::memset(data.data(), 0, data.size() * sizeof(T)); }
};
using VectorBatch64 = VectorBatch<double>;
using VectorBatch32 = VectorBatch<float>;

// ------------------------------------------------------- solution_io.hpp:12-84
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

template <typename T>
struct BlockJacobi {  // block_jacobi.hpp:15-39 (host copy of the inverse blocks)
  std::vector<std::array<T, 9>> inv_blocks;
  int32_t n_nodes() const { return static_cast<int32_t>(inv_blocks.size()); }
};

// ----------------------------------------------------- ebe_operator.hpp:29-226
template <typename T>
class EbeOperator {
 public:
  EbeOperator() = default;
  // EbeOperator(mesh, order, materials, dof_mask, workers) (ebe_operator.hpp:35-36);
  // `workers` is accepted and ignored: the device sweep is order-independent.
  EbeOperator(const Mesh& mesh, int order, const std::vector<Material>& materials, std::vector<uint8_t> dof_mask,
              int workers = 1)
      : order_(order), mask_(std::move(dof_mask)) {
    (void)workers;
    detail::MeshHandle mh(mesh);
    auto [l, m] = detail::lame(materials);
    ts_ebe* h = nullptr;
    detail::check(ts_ebe_create(mh.h, order, static_cast<int32_t>(l.size()), l.data(), m.data(),
                                mask_.empty() ? nullptr : mask_.data(), sizeof(T) == 4 ? 32 : 64, &h));
    op_ = std::shared_ptr<ts_ebe>(h, ts_ebe_destroy);
    int32_t nn, ne;
    ts_ebe_info(h, &nn, &ne, nullptr, nullptr);
    n_nodes_ = nn;
    n_elems_ = ne;
    conn_.resize(static_cast<size_t>(nodes_per_element()) * ne);
    for (int32_t e = 0; e < ne; ++e)
      for (int a = 0; a < nodes_per_element(); ++a)
        conn_[static_cast<size_t>(nodes_per_element()) * e + a] = mesh.tets10[e][a];
  }
  // non-owning view of an operator inside a SolverLevels
  EbeOperator(std::shared_ptr<ts_ebe> op, int32_t n_nodes, int32_t n_elems, int order)
      : op_(std::move(op)), order_(order), n_nodes_(n_nodes), n_elems_(n_elems) {}

  int32_t n_nodes() const { return n_nodes_; }
  int32_t n_elements() const { return n_elems_; }
  int order() const { return order_; }
  int nodes_per_element() const { return order_ == 1 ? 4 : 10; }
  const std::vector<uint8_t>& mask() const { return mask_; }
  int32_t element_node(int32_t e, int a) const { return conn_[static_cast<size_t>(nodes_per_element()) * e + a]; }

  // f = A u for all batch columns (ebe_operator.hpp:90-134): host buffers in/out
  void apply(const VectorBatch<T>& u, VectorBatch<T>& f) const {
    if (u.n_nodes != n_nodes_) throw ValidationError("ebe apply: dimension mismatch");
    if (f.n_nodes != u.n_nodes || f.batch != u.batch) f = VectorBatch<T>(u.n_nodes, u.batch);
    detail::check(ts_ebe_apply_host(op_.get(), u.data.data(), f.data.data(), u.batch));
  }
  // device-pointer entry for callers that keep vectors in HBM
  void apply_device(const T* u, T* f, int32_t batch, void* stream = nullptr) const {
    detail::check(ts_ebe_apply(op_.get(), u, f, batch, stream));
  }
  const ts_ebe* handle() const { return op_.get(); }

 private:
  std::shared_ptr<ts_ebe> op_;
  int order_ = 2;
  int32_t n_nodes_ = 0, n_elems_ = 0;
  std::vector<uint8_t> mask_;
  std::vector<int32_t> conn_;
};

// extract_block_jacobi(EbeOperator) (ebe_operator.hpp:288-313), computed on the GPU
template <typename T>
inline BlockJacobi<T> extract_block_jacobi(const EbeOperator<T>& op) {
  BlockJacobi<T> m;
  m.inv_blocks.resize(op.n_nodes());
  detail::check(ts_ebe_block_jacobi_host(op.handle(), m.inv_blocks.data()));
  return m;
}

// ------------------------------------------------------ adaptive_cg.hpp:27-67
class SolverLevels {
 public:
  SolverLevels() = default;
  explicit SolverLevels(ts_levels* h) : SolverLevels(std::shared_ptr<ts_levels>(h, ts_levels_destroy)) {}
  // a level set owned elsewhere (e.g. by a faulted model): `lv` shares the owner's lifetime
  explicit SolverLevels(std::shared_ptr<ts_levels> lv) : lv_(std::move(lv)) {
    ts_levels* h = lv_.get();
    int32_t n0, n1, n2;
    ts_levels_sizes(h, &n0, &n1, &n2, nullptr);
    const ts_ebe* o;
    ts_levels_operator(h, 0, &o);
    int32_t ne;
    ts_ebe_info(o, nullptr, &ne, nullptr, nullptr);
    // operators are owned by the level set; views share its lifetime
    auto keep = lv_;
    auto view = [&](int which) {
      const ts_ebe* p;
      ts_levels_operator(h, which, &p);
      return std::shared_ptr<ts_ebe>(keep, const_cast<ts_ebe*>(p));
    };
    outer = EbeOperator<double>(view(0), n0, ne, 2);
    level0 = EbeOperator<float>(view(1), n0, ne, 2);
    level1 = EbeOperator<float>(view(2), n1, ne, 1);
    n2_ = n2;
  }
  EbeOperator<double> outer;
  EbeOperator<float> level0, level1;
  int32_t level2_rows() const { return n2_; }
  ts_levels* handle() const { return lv_.get(); }

 private:
  std::shared_ptr<ts_levels> lv_;
  int32_t n2_ = 0;
};

inline SolverLevels build_solver_levels(const Mesh& mesh, const std::vector<Material>& materials,
                                        const std::vector<uint8_t>& dof_mask, const SolverConfig& cfg,
                                        int workers = 1) {
  (void)workers;
  detail::MeshHandle mh(mesh);
  auto [l, m] = detail::lame(materials);
  const ts_solver_config c = cfg.to_c();
  ts_levels* h = nullptr;
  detail::check(ts_levels_create(mh.h, static_cast<int32_t>(l.size()), l.data(), m.data(),
                                 dof_mask.empty() ? nullptr : dof_mask.data(), &c, &h));
  return SolverLevels(h);
}

struct CrustModel {  // model.hpp:14-19
  Mesh mesh;
  std::vector<Material> materials;
  std::vector<uint8_t> mask;
  SolverLevels levels;
};

inline CrustModel build_crust_model(Mesh mesh, std::vector<Material> materials, const SolverConfig& cfg,
                                    int workers = 1) {  // model.hpp:21-29
  CrustModel model;
  model.mask = dirichlet_mask(mesh);
  model.levels = build_solver_levels(mesh, materials, model.mask, cfg, workers);
  model.mesh = std::move(mesh);
  model.materials = std::move(materials);
  return model;
}

namespace detail {
struct ReportBuf {
  ts_solve_report c{};
  std::vector<double> final_, hist;
  std::vector<int32_t> hit;
  ReportBuf(int32_t batch, int32_t cap) : final_(batch), hist(size_t(cap > 0 ? cap : 1) * batch), hit(cap > 0 ? cap : 1) {
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

// solve (adaptive_cg.hpp:242-263): host VectorBatch in/out, GPU inside
inline std::pair<VectorBatch64, SolveReport> solve(const SolverLevels& levels, const VectorBatch64& f,
                                                   const VectorBatch64& u0, const SolverConfig& cfg) {
  if (u0.n_nodes != f.n_nodes || u0.batch != f.batch) throw ValidationError("solve: initial guess shape mismatch");
  const ts_solver_config c = cfg.to_c();
  const int32_t cap = cfg.residual_history_stride > 0 ? cfg.outer_max_iter / cfg.residual_history_stride + 1 : 0;
  detail::ReportBuf rb(f.batch, cap);
  VectorBatch64 u(f.n_nodes, f.batch);
  detail::finish(ts_solve(levels.handle(), f.data.data(), u0.data.data(), u.data.data(), f.batch, &c, &rb.c), rb,
                 cfg.residual_history_stride);
  return {std::move(u), rb.report(cfg.residual_history_stride)};
}

// solve_pcge (adaptive_cg.hpp:267-279)
inline std::pair<VectorBatch64, SolveReport> solve_pcge(const EbeOperator<double>& k, const VectorBatch64& f,
                                                        const VectorBatch64& u0, double tol, int max_iter) {
  detail::ReportBuf rb(f.batch, 0);
  VectorBatch64 u(f.n_nodes, f.batch);
  detail::finish(ts_solve_pcge(k.handle(), f.data.data(), u0.data.data(), u.data.data(), f.batch, tol, max_iter,
                               &rb.c),
                 rb, 0);
  return {std::move(u), rb.report(0)};
}

// ------------------------------------------- fault.hpp / model.hpp / greens.hpp
// The Green's-function sweep. Split-node geometry, slip
// lifting, the batched solves and the sampling run inside the library; the
// types keep the reference's names and fields so a sweep written against
// tetsolve compiles unchanged (FaultPatch is a summary: its geometry stays in
// the library, and UnitSlip magnitudes are evaluated there).
enum class SlipDirection { dip = 0, strike = 1 };  // fault.hpp:12-15

struct ObservationComponent {  // greens.hpp:15-18
  Vec3 point{};
  int axis = 0;
};

struct FaultPatch {  // fault.hpp:37-41 (summary)
  int32_t n_faces = 0;
  int32_t n_split_nodes = 0;
};

struct UnitSlip {  // fault.hpp:308-315
  Vec3 center{};
  SlipDirection direction = SlipDirection::dip;
  double radius = 0.0;
  std::vector<double> magnitude;  // evaluated by the library (unit_slip_magnitudes)
};

struct FaultedModel {  // model.hpp:34-39
  CrustModel base;
  FaultPatch patch;
  int32_t split_mesh_nodes = 0;
  std::shared_ptr<ts_faulted> handle;
};

// find_plane_fault_faces (fault.hpp:86-118)
inline std::vector<std::array<int32_t, 3>> find_plane_fault_faces(const Mesh& mesh, int axis, double coord,
                                                                  const Vec3& lo, const Vec3& hi) {
  detail::MeshHandle h(mesh);
  int32_t n = 0;
  detail::check(ts_fault_plane_faces(h.h, axis, coord, lo.data(), hi.data(), &n, nullptr));
  std::vector<std::array<int32_t, 3>> faces(n);
  if (n) detail::check(ts_fault_plane_faces(h.h, axis, coord, lo.data(), hi.data(), &n, faces[0].data()));
  return faces;
}

// build_faulted_model (model.hpp:41-51)
inline FaultedModel build_faulted_model(Mesh mesh, std::vector<Material> materials,
                                        const std::vector<std::array<int32_t, 3>>& fault_tris,
                                        const SolverConfig& cfg, int /*workers*/ = 1) {
  detail::MeshHandle h(mesh);
  const auto [lam, mu] = detail::lame(materials);
  const ts_solver_config c = cfg.to_c();
  ts_faulted* f = nullptr;
  detail::check(ts_faulted_model_create(h.h, static_cast<int32_t>(materials.size()), lam.data(), mu.data(),
                                        fault_tris.empty() ? nullptr : fault_tris[0].data(),
                                        static_cast<int32_t>(fault_tris.size()), &c, &f));
  FaultedModel fm;
  fm.handle = std::shared_ptr<ts_faulted>(f, ts_faulted_model_destroy);
  detail::check(ts_faulted_info(f, &fm.patch.n_split_nodes, &fm.split_mesh_nodes, &fm.patch.n_faces));
  ts_levels* lv = nullptr;
  detail::check(ts_faulted_levels(f, &lv));
  fm.base.mask = dirichlet_mask(mesh);
  fm.base.levels = SolverLevels(std::shared_ptr<ts_levels>(fm.handle, lv));
  fm.base.mesh = std::move(mesh);
  fm.base.materials = std::move(materials);
  return fm;
}

// unit_slip_basis (fault.hpp:325-343): the magnitudes are evaluated in the library
inline UnitSlip unit_slip_basis(const FaultPatch& patch, const Mesh& /*base_mesh*/, const Vec3& center,
                                SlipDirection direction, double radius) {
  if (radius <= 0.0) throw ValidationError("unit_slip_basis: radius must be positive");
  if (patch.n_faces == 0) throw ValidationError("unit_slip_basis: empty fault patch");
  UnitSlip s;
  s.center = center;
  s.direction = direction;
  s.radius = radius;
  return s;
}

namespace detail {
struct SlipArrays {
  std::vector<double> centers, radii;
  std::vector<int32_t> dirs;
  explicit SlipArrays(const std::vector<UnitSlip>& slips) {
    for (const auto& s : slips) {
      centers.insert(centers.end(), s.center.begin(), s.center.end());
      dirs.push_back(static_cast<int32_t>(s.direction));
      radii.push_back(s.radius);
    }
  }
};
}  // namespace detail

// slip_to_rhs (model.hpp:53-56)
inline VectorBatch64 slip_to_rhs(const FaultedModel& fm, const UnitSlip& slip) {
  const detail::SlipArrays a({slip});
  VectorBatch64 f(fm.base.mesh.node_count(), 1);
  detail::check(ts_slip_to_rhs(fm.handle.get(), 1, a.centers.data(), a.dirs.data(), a.radii.data(), f.data.data()));
  return f;
}

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

// Green's-sweep files (fault.hpp:44-84,414-419; greens.hpp:20-44,147-222): the reference's bytes
inline void write_fault_faces(const std::vector<std::array<int32_t, 3>>& faces, const std::string& path) {
  detail::check(ts_fault_faces_write(path.c_str(), faces.empty() ? nullptr : faces[0].data(),
                                     static_cast<int32_t>(faces.size())));
}
inline std::vector<std::array<int32_t, 3>> read_fault_faces(const std::string& path) {
  int32_t n = 0;
  detail::check(ts_fault_faces_read(path.c_str(), &n, nullptr));
  std::vector<std::array<int32_t, 3>> f(n);
  detail::check(ts_fault_faces_read(path.c_str(), &n, f.empty() ? nullptr : f[0].data()));
  return f;
}
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
