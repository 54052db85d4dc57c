// abi.cpp — extern "C" boundary of libtsgpu.so (include/tsgpu.h): argument
// validation, exception -> ts_status translation, host-buffer conveniences.
#include <array>
#include <cstring>
#include <memory>

#include "comm.h"
#include "dist.h"
#include "dist_api.h"
#include "ebe.h"
#include "mesh_io.h"
#include "setup.h"

namespace tsg {
const std::string& last_error();
}

#define TS_API_BEGIN try {
#define TS_API_END                                                  \
  }                                                                 \
  catch (const tsg::Error& e) {                                     \
    tsg::set_last_error(e.what());                                  \
    return e.code;                                                  \
  }                                                                 \
  catch (const std::bad_alloc&) {                                   \
    tsg::set_last_error("out of host memory");                      \
    return TS_ERR_VALIDATION;                                       \
  }                                                                 \
  catch (const std::exception& e) {                                 \
    tsg::set_last_error(e.what());                                  \
    return TS_ERR_VALIDATION;                                       \
  }                                                                 \
  return TS_OK;

// a partitioned call that fails on one rank aborts the communicator, so peers
// blocked in (or entering) a collective fail instead of waiting forever. The
// solver's own outcomes (no convergence, breakdown, non-finite residual) are
// decided on all-reduced numbers, so every rank reaches them at the same point:
// they end the call on all ranks together and leave the communicator usable.
#define TS_ABORT_ON_FAIL(comm, ...)                                              \
  try {                                                                          \
    __VA_ARGS__;                                                                 \
  } catch (const tsg::Error& e_) {                                               \
    if ((comm) && e_.code != TS_ERR_NO_CONVERGENCE && e_.code != TS_ERR_BREAKDOWN && \
        e_.code != TS_ERR_NONFINITE)                                             \
      (comm)->abort();                                                           \
    throw;                                                                       \
  } catch (...) {                                                                \
    if (comm) (comm)->abort();                                                   \
    throw;                                                                       \
  }

#define TS_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) tsg::validation(msg); \
  } while (0)

struct ts_comm {
  std::unique_ptr<tsg::Comm> c;
};
tsg::Comm* tsg::comm_of(ts_comm* c) { return c ? c->c.get() : nullptr; }
struct ts_thread_world {
  std::shared_ptr<tsg::ThreadWorld> w;
};

extern "C" {

const char* ts_last_error(void) { return tsg::last_error().c_str(); }
const char* ts_version(void) { return "tsgpu 0.1 (sm_100a)"; }

void ts_config_default(ts_solver_config* c) {
  if (!c) return;
  c->outer_tol = 1e-8;
  c->outer_max_iter = 5000;
  c->level_tol[0] = 0.1;
  c->level_tol[1] = 0.05;
  c->level_tol[2] = 0.025;
  c->level_max_iter[0] = 30;
  c->level_max_iter[1] = 300;
  c->level_max_iter[2] = 3000;
  c->batch_size = 16;
  c->aggregate_target = 8;
  c->residual_history_stride = 1;
}

ts_status ts_config_validate(const ts_solver_config* c) {
  TS_API_BEGIN
  TS_REQUIRE(c, "solver config: null");
  auto check_tol = [](double t, const char* what) {
    if (!(t > 0.0 && t < 1.0))
      tsg::validation(std::string("solver config: ") + what + " tolerance must lie in (0, 1)");
  };
  check_tol(c->outer_tol, "outer");
  check_tol(c->level_tol[0], "level 0");
  check_tol(c->level_tol[1], "level 1");
  check_tol(c->level_tol[2], "level 2");
  if (c->outer_max_iter < 1 || c->level_max_iter[0] < 1 || c->level_max_iter[1] < 1 ||
      c->level_max_iter[2] < 1)
    tsg::validation("solver config: max iterations must be >= 1");
  if (c->batch_size < 1) tsg::validation("solver config: batch size must be >= 1");
  if (c->aggregate_target < 2) tsg::validation("solver config: aggregate target must be >= 2");
  TS_API_END
}

// ------------------------------------------------------------------- mesh
ts_status ts_box_mesh(const double extents[3], const int32_t divisions[3], int32_t n_interfaces,
                      const double* layer_interfaces, int32_t fixed_boundary, ts_mesh** out) {
  TS_API_BEGIN
  TS_REQUIRE(extents && divisions && out, "box mesh: null argument");
  TS_REQUIRE(fixed_boundary >= 0 && fixed_boundary <= 2, "box mesh: fixed_boundary must be 0, 1 or 2");
  std::vector<double> ifs;
  if (n_interfaces > 0) ifs.assign(layer_interfaces, layer_interfaces + n_interfaces);
  auto h = std::make_unique<ts_mesh>();
  h->m = tsg::generate_box_mesh(extents, divisions, ifs, fixed_boundary);
  *out = h.release();
  TS_API_END
}

ts_status ts_mesh_from_arrays(int32_t n_nodes, int32_t vertex_count, const double* coords,
                              int32_t n_elems, const int32_t* tets10, const int32_t* material_id,
                              int32_t n_dirichlet, const int32_t* bc_node, const int8_t* bc_axis,
                              ts_mesh** out) {
  TS_API_BEGIN
  TS_REQUIRE(out && n_nodes >= 0 && n_elems >= 0 && vertex_count >= 0 && vertex_count <= n_nodes,
             "mesh: bad sizes");
  TS_REQUIRE((n_nodes == 0 || coords) && (n_elems == 0 || (tets10 && material_id)),
             "mesh: null array");
  auto h = std::make_unique<ts_mesh>();
  auto& m = h->m;
  m.coords.assign(coords, coords + 3 * static_cast<size_t>(n_nodes));
  m.tets10.assign(tets10, tets10 + 10 * static_cast<size_t>(n_elems));
  m.material_id.assign(material_id, material_id + n_elems);
  m.vertex_count = vertex_count;
  for (int32_t i = 0; i < n_dirichlet; ++i) {
    TS_REQUIRE(bc_node[i] >= 0 && bc_node[i] < n_nodes && bc_axis[i] >= 0 && bc_axis[i] <= 2,
               "mesh: dirichlet entry out of range");
    m.bc_node.push_back(bc_node[i]);
    m.bc_axis.push_back(bc_axis[i]);
  }
  for (size_t q = 0; q < m.tets10.size(); ++q)
    TS_REQUIRE(m.tets10[q] >= 0 && m.tets10[q] < n_nodes,
               "mesh: element " + std::to_string(q / 10) + " references node " +
                   std::to_string(m.tets10[q]) + " out of range");
  *out = h.release();
  TS_API_END
}

ts_status ts_mesh_validate(const ts_mesh* m) {
  TS_API_BEGIN
  TS_REQUIRE(m, "mesh: null handle");
  tsg::validate_mesh(m->m);
  TS_API_END
}

// ------------------------------------------------------------ file formats
ts_status ts_mesh_write_tsmesh(const ts_mesh* m, const char* path) {
  TS_API_BEGIN
  TS_REQUIRE(m && path, "mesh io: null argument");
  tsg::write_tsmesh(m->m, path);
  TS_API_END
}

ts_status ts_mesh_read_tsmesh(const char* path, ts_mesh** out) {
  TS_API_BEGIN
  TS_REQUIRE(path && out, "mesh io: null argument");
  auto h = std::make_unique<ts_mesh>();
  h->m = tsg::read_tsmesh(path);
  *out = h.release();
  TS_API_END
}

ts_status ts_mesh_write_dirichlet(const ts_mesh* m, const char* path) {
  TS_API_BEGIN
  TS_REQUIRE(m && path, "mesh io: null argument");
  tsg::write_dirichlet(m->m, path);
  TS_API_END
}

ts_status ts_mesh_read_dirichlet(ts_mesh* m, const char* path) {
  TS_API_BEGIN
  TS_REQUIRE(m && path, "mesh io: null argument");
  tsg::read_dirichlet(m->m, path);
  TS_API_END
}

ts_status ts_mesh_write_tsbmesh(const ts_mesh* m, const char* path) {
  TS_API_BEGIN
  TS_REQUIRE(m && path, "mesh io: null argument");
  tsg::write_tsbmesh(m->m, path);
  TS_API_END
}

ts_status ts_mesh_read_tsbmesh(const char* path, ts_mesh** out) {
  TS_API_BEGIN
  TS_REQUIRE(path && out, "mesh io: null argument");
  auto h = std::make_unique<ts_mesh>();
  h->m = tsg::read_tsbmesh(path);
  *out = h.release();
  TS_API_END
}

ts_status ts_tsvec_write(const char* path, const double* u, int64_t nodes, int32_t batch, int32_t on_device) {
  TS_API_BEGIN
  TS_REQUIRE(path && (u || nodes == 0), "solution io: null argument");
  tsg::write_tsvec(path, u, nodes, batch, on_device != 0);
  TS_API_END
}

ts_status ts_tsvec_info(const char* path, int64_t* nodes, int32_t* batch) {
  TS_API_BEGIN
  TS_REQUIRE(path, "solution io: null argument");
  int64_t n, b, off;
  tsg::tsvec_info(path, &n, &b, &off);
  TS_REQUIRE(b <= INT32_MAX, "solution io: batch out of range");
  if (nodes) *nodes = n;
  if (batch) *batch = static_cast<int32_t>(b);
  TS_API_END
}

ts_status ts_tsvec_read(const char* path, double* u, int64_t nodes, int32_t batch, int32_t on_device) {
  TS_API_BEGIN
  TS_REQUIRE(path && (u || nodes == 0), "solution io: null argument");
  tsg::read_tsvec(path, u, nodes, batch, on_device != 0);
  TS_API_END
}

// ------------------------------------------------------------ Green's-sweep files
ts_status ts_fault_faces_write(const char* path, const int32_t* faces, int32_t n) {
  TS_API_BEGIN
  TS_REQUIRE(path && n >= 0 && (faces || n == 0), "fault file: bad argument");
  std::vector<std::array<int32_t, 3>> f(static_cast<size_t>(n));
  if (n) std::memcpy(f.data(), faces, sizeof(int32_t) * 3 * size_t(n));
  tsg::write_fault_faces(f, path);
  TS_API_END
}

ts_status ts_fault_faces_read(const char* path, int32_t* n, int32_t* faces) {
  TS_API_BEGIN
  TS_REQUIRE(path && n, "fault file: null argument");
  const auto f = tsg::read_fault_faces(path);
  if (faces) {
    TS_REQUIRE(*n >= static_cast<int32_t>(f.size()), "fault file: output too small");
    std::memcpy(faces, f.data(), sizeof(int32_t) * 3 * f.size());
  }
  *n = static_cast<int32_t>(f.size());
  TS_API_END
}

ts_status ts_observations_read(const char* path, int32_t* n, double* points, int32_t* axes) {
  TS_API_BEGIN
  TS_REQUIRE(path && n, "observations: null argument");
  const auto o = tsg::read_observations(path);
  if (points || axes) {
    TS_REQUIRE(*n >= static_cast<int32_t>(o.size()), "observations: output too small");
    for (size_t i = 0; i < o.size(); ++i) {
      if (points)
        for (int c = 0; c < 3; ++c) points[3 * i + c] = o[i].p[c];
      if (axes) axes[i] = o[i].axis;
    }
  }
  *n = static_cast<int32_t>(o.size());
  TS_API_END
}

ts_status ts_greens_bank_write(const char* path, int32_t rows, int32_t cols, const double* obs_points,
                               const int32_t* obs_axes, const double* centers, const int32_t* directions,
                               const double* radii, const double* values) {
  TS_API_BEGIN
  TS_REQUIRE(path && rows >= 1 && cols >= 1 && obs_points && obs_axes && centers && directions && radii && values,
             "greens bank: bad argument");
  tsg::GreensBankData g;
  g.rows = rows;
  g.cols = cols;
  for (int32_t r = 0; r < rows; ++r) {
    tsg::Observation o;
    for (int c = 0; c < 3; ++c) o.p[c] = obs_points[3 * r + c];
    o.axis = obs_axes[r];
    g.obs.push_back(o);
  }
  g.centers.assign(centers, centers + 3 * size_t(cols));
  g.dirs.assign(directions, directions + cols);
  g.radii.assign(radii, radii + cols);
  g.values.assign(values, values + size_t(rows) * cols);
  tsg::write_greens_bank(g, path);
  TS_API_END
}

ts_status ts_greens_bank_read(const char* path, int32_t* rows, int32_t* cols, double* obs_points, int32_t* obs_axes,
                              double* centers, int32_t* directions, double* radii, double* values) {
  TS_API_BEGIN
  TS_REQUIRE(path && rows && cols, "greens bank: null argument");
  const tsg::GreensBankData g = tsg::read_greens_bank(path);
  const bool fill = obs_points || obs_axes || centers || directions || radii || values;
  if (fill) TS_REQUIRE(*rows >= g.rows && *cols >= g.cols, "greens bank: output too small");
  *rows = g.rows;
  *cols = g.cols;
  for (int32_t r = 0; fill && r < g.rows; ++r) {
    if (obs_points)
      for (int c = 0; c < 3; ++c) obs_points[3 * r + c] = g.obs[r].p[c];
    if (obs_axes) obs_axes[r] = g.obs[r].axis;
  }
  if (centers) std::copy(g.centers.begin(), g.centers.end(), centers);
  if (directions) std::copy(g.dirs.begin(), g.dirs.end(), directions);
  if (radii) std::copy(g.radii.begin(), g.radii.end(), radii);
  if (values) std::copy(g.values.begin(), g.values.end(), values);
  TS_API_END
}

ts_status ts_mesh_sizes(const ts_mesh* h, int32_t* nn, int32_t* nv, int32_t* ne, int32_t* nbc) {
  TS_API_BEGIN
  TS_REQUIRE(h, "mesh: null handle");
  if (nn) *nn = h->m.n_nodes();
  if (nv) *nv = h->m.vertex_count;
  if (ne) *ne = h->m.n_elems();
  if (nbc) *nbc = static_cast<int32_t>(h->m.bc_node.size());
  TS_API_END
}

ts_status ts_mesh_export(const ts_mesh* h, double* coords, int32_t* tets10, int32_t* material_id,
                         int32_t* bc_node, int8_t* bc_axis) {
  TS_API_BEGIN
  TS_REQUIRE(h, "mesh: null handle");
  const auto& m = h->m;
  if (coords) std::memcpy(coords, m.coords.data(), m.coords.size() * sizeof(double));
  if (tets10) std::memcpy(tets10, m.tets10.data(), m.tets10.size() * sizeof(int32_t));
  if (material_id) std::memcpy(material_id, m.material_id.data(), m.material_id.size() * sizeof(int32_t));
  if (bc_node) std::memcpy(bc_node, m.bc_node.data(), m.bc_node.size() * sizeof(int32_t));
  if (bc_axis) std::memcpy(bc_axis, m.bc_axis.data(), m.bc_axis.size());
  TS_API_END
}

ts_status ts_mesh_dirichlet_mask(const ts_mesh* h, uint8_t* mask) {
  TS_API_BEGIN
  TS_REQUIRE(h && mask, "mesh: null argument");
  const auto v = h->m.dirichlet_mask();
  std::memcpy(mask, v.data(), v.size());
  TS_API_END
}

void ts_mesh_destroy(ts_mesh* m) { delete m; }

ts_status ts_material_from_wavespeeds(double vp, double vs, double rho, double* lambda, double* mu) {
  TS_API_BEGIN
  TS_REQUIRE(lambda && mu, "material: null output");
  if (vp <= 0.0 || vs <= 0.0 || rho <= 0.0) tsg::validation("material: vp, vs, rho must be positive");
  if (vp * vp <= 2.0 * vs * vs)
    tsg::validation("material: requires vp^2 > 2*vs^2 (lambda must be positive)");
  *mu = rho * vs * vs;
  *lambda = rho * (vp * vp - 2.0 * vs * vs);
  TS_API_END
}

// ------------------------------------------------------------------- EBE
ts_status ts_ebe_create(const ts_mesh* mesh, int32_t order, int32_t n_materials,
                        const double* lambda, const double* mu, const uint8_t* dof_mask,
                        int32_t prec, ts_ebe** out) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && out && lambda && mu && n_materials >= 0, "ebe: null argument");
  *out = tsg::ebe_create(mesh->m, order, n_materials, lambda, mu, dof_mask, prec);
  TS_API_END
}

void ts_ebe_destroy(ts_ebe* op) { delete op; }

ts_status ts_ebe_info(const ts_ebe* op, int32_t* n_nodes, int32_t* n_elements, int32_t* order,
                      int32_t* prec) {
  TS_API_BEGIN
  TS_REQUIRE(op, "ebe: null handle");
  if (n_nodes) *n_nodes = op->n_nodes;
  if (n_elements) *n_elements = op->n_elems;
  if (order) *order = op->order;
  if (prec) *prec = op->prec;
  TS_API_END
}

ts_status ts_ebe_apply(const ts_ebe* op, const void* u, void* f, int32_t batch, void* stream) {
  TS_API_BEGIN
  TS_REQUIRE(op && u && f, "ebe apply: null argument");
  tsg::ebe_apply(*op, u, f, batch, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_ebe_apply_host(const ts_ebe* op, const void* u, void* f, int32_t batch) {
  TS_API_BEGIN
  TS_REQUIRE(op && u && f, "ebe apply: null argument");
  TS_REQUIRE(batch >= 1, "ebe apply: batch must be >= 1");
  tsg::ebe_apply_host(*op, u, f, batch);
  TS_API_END
}

ts_status ts_ebe_host_stream_chunks(const ts_ebe* op, int32_t* chunks) {
  TS_API_BEGIN
  TS_REQUIRE(op && chunks, "ebe: null argument");
  std::lock_guard<std::mutex> lock(op->host_mu);
  *chunks = op->stream && op->stream->usable ? op->stream->chunks : 0;
  TS_API_END
}

ts_status ts_ebe_block_jacobi_host(const ts_ebe* op, void* inv_blocks) {
  TS_API_BEGIN
  TS_REQUIRE(op && inv_blocks, "ebe block jacobi: null argument");
  const size_t bytes = 9 * static_cast<size_t>(op->n_nodes) * (op->prec / 8);
  tsg::DevBuf<unsigned char> d(bytes);
  tsg::ebe_block_jacobi(*op, d.get(), nullptr);
  TS_CUDA(cudaMemcpy(inv_blocks, d.get(), bytes, cudaMemcpyDeviceToHost));
  TS_API_END
}

ts_status ts_ebe_set_timing(ts_ebe* op, int32_t enable) {
  TS_API_BEGIN
  TS_REQUIRE(op, "ebe: null handle");
  if (enable && !op->ev0) {
    TS_CUDA(cudaEventCreate(&op->ev0));
    TS_CUDA(cudaEventCreate(&op->ev1));
  }
  op->timing = enable != 0;
  TS_API_END
}

ts_status ts_ebe_last_kernel_ms(const ts_ebe* op, float* ms) {
  TS_API_BEGIN
  TS_REQUIRE(op && ms, "ebe: null argument");
  TS_REQUIRE(op->timing, "ebe: timing not enabled");
  TS_CUDA(cudaEventSynchronize(op->ev1));
  TS_CUDA(cudaEventElapsedTime(ms, op->ev0, op->ev1));
  TS_API_END
}

ts_status ts_ebe_set_deterministic(ts_ebe* op, int32_t on) {
  TS_API_BEGIN
  TS_REQUIRE(op, "ebe: null handle");
  tsg::ebe_set_deterministic(*op, on != 0);
  TS_API_END
}

ts_status ts_ebe_launches_per_apply(const ts_ebe* op, int32_t batch, int32_t* n) {
  TS_API_BEGIN
  TS_REQUIRE(op && n, "ebe: null argument");
  TS_REQUIRE(batch >= 1, "ebe: batch must be >= 1");
  *n = tsg::ebe_launches_per_apply(*op, batch);
  TS_API_END
}

ts_status ts_ebe_unit_stats(const ts_ebe* op, int32_t* kind, int32_t* units, double* rows_per_element,
                            double* closed_fraction, double* elements_per_unit) {
  TS_API_BEGIN
  TS_REQUIRE(op && kind && units && rows_per_element && closed_fraction && elements_per_unit, "ebe: null argument");
  if (op->fan) {
    *kind = 2;
    *units = op->fan->n_units;
    *rows_per_element = op->fan->rows_per_element;
    *closed_fraction = op->fan->closed_fraction;
    *elements_per_unit = op->fan->mean_k;
  } else if (op->pair) {
    *kind = 1;
    *units = op->pair->n_units;
    const double pf = op->pair->paired_fraction;
    const int npe = op->npe, nr = npe == 10 ? 14 : 5;
    *rows_per_element = pf * nr / 2.0 + (1.0 - pf) * npe;
    *closed_fraction = pf;
    *elements_per_unit = op->pair->n_units ? double(op->n_elems) / op->pair->n_units : 0.0;
  } else {
    *kind = 0;
    *units = op->n_elems;
    *rows_per_element = op->npe;
    *closed_fraction = 0.0;
    *elements_per_unit = 1.0;
  }
  TS_API_END
}

// ------------------------------------------------------------ partitioned solve
ts_status ts_comm_nccl_available(char* why, int32_t why_len) {
  TS_API_BEGIN
  std::string w;
  const bool ok = tsg::nccl_available(&w);
  if (why && why_len > 0) {
    std::strncpy(why, w.c_str(), size_t(why_len) - 1);
    why[why_len - 1] = 0;
  }
  if (!ok) tsg::fail(TS_ERR_NCCL, "nccl unavailable: " + w);
  TS_API_END
}

ts_status ts_comm_nccl_id(uint8_t id[128]) {
  TS_API_BEGIN
  TS_REQUIRE(id, "comm: null id");
  tsg::nccl_unique_id(id);
  TS_API_END
}

ts_status ts_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device, ts_comm** out) {
  TS_API_BEGIN
  TS_REQUIRE(id && out, "comm: null argument");
  auto h = std::make_unique<ts_comm>();
  h->c = tsg::make_nccl_comm(nranks, rank, id, device);
  *out = h.release();
  TS_API_END
}

ts_status ts_thread_world_create(int32_t nranks, ts_thread_world** out) {
  TS_API_BEGIN
  TS_REQUIRE(out, "comm: null argument");
  auto h = std::make_unique<ts_thread_world>();
  h->w = tsg::make_thread_world(nranks);
  *out = h.release();
  TS_API_END
}

void ts_thread_world_destroy(ts_thread_world* w) { delete w; }

ts_status ts_comm_create_thread(ts_thread_world* w, int32_t rank, int32_t device, ts_comm** out) {
  TS_API_BEGIN
  TS_REQUIRE(w && out, "comm: null argument");
  auto h = std::make_unique<ts_comm>();
  h->c = tsg::make_thread_comm(w->w, rank, device);
  *out = h.release();
  TS_API_END
}

void ts_comm_destroy(ts_comm* c) { delete c; }

ts_status ts_comm_info(const ts_comm* c, int32_t* rank, int32_t* size, int32_t* device) {
  TS_API_BEGIN
  TS_REQUIRE(c, "comm: null handle");
  if (rank) *rank = c->c->rank();
  if (size) *size = c->c->size();
  if (device) *device = c->c->device();
  TS_API_END
}

ts_status ts_comm_allreduce_sum(const ts_comm* c, double* data, int64_t n, void* stream) {
  TS_API_BEGIN
  TS_REQUIRE(c && (data || n == 0) && n >= 0, "comm allreduce: bad argument");
  if (n > 0) c->c->allreduce_sum(data, static_cast<size_t>(n), static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_partition_rcb(const ts_mesh* mesh, int32_t nparts, int32_t* part) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && part, "partition: null argument");
  const std::vector<int32_t> p = tsg::partition_rcb(mesh->m, nparts);
  std::memcpy(part, p.data(), p.size() * sizeof(int32_t));
  TS_API_END
}

ts_status ts_dist_plan_sizes(const ts_mesh* mesh, const uint8_t* dof_mask, const int32_t* part, int32_t nranks,
                             int32_t rank, int32_t* n_local, int32_t* n_local_vertices, int32_t* n_elems,
                             int32_t* n_nbr, int64_t* n_halo_rows) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && part, "dist plan: null argument");
  const tsg::DistPlan p = tsg::build_dist_plan(mesh->m, dof_mask, part, nranks, rank);
  if (n_local) *n_local = p.n_local;
  if (n_local_vertices) *n_local_vertices = p.n_local_vertices;
  if (n_elems) *n_elems = static_cast<int32_t>(p.elems.size());
  if (n_nbr) *n_nbr = static_cast<int32_t>(p.halo0.nbr.size());
  if (n_halo_rows) *n_halo_rows = p.halo0.rows_total();
  TS_API_END
}

ts_status ts_dist_plan_export(const ts_mesh* mesh, const uint8_t* dof_mask, const int32_t* part, int32_t nranks,
                              int32_t rank, int32_t* l2g, uint8_t* owned, int32_t* elems, int32_t* nbr,
                              int32_t* nbr_rows, int32_t* halo_rows) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && part, "dist plan: null argument");
  const tsg::DistPlan p = tsg::build_dist_plan(mesh->m, dof_mask, part, nranks, rank);
  if (l2g) std::memcpy(l2g, p.l2g.data(), p.l2g.size() * sizeof(int32_t));
  if (owned) std::memcpy(owned, p.owned.data(), p.owned.size());
  if (elems) std::memcpy(elems, p.elems.data(), p.elems.size() * sizeof(int32_t));
  int64_t o = 0;
  for (size_t k = 0; k < p.halo0.nbr.size(); ++k) {
    if (nbr) nbr[k] = p.halo0.nbr[k];
    if (nbr_rows) nbr_rows[k] = static_cast<int32_t>(p.halo0.rows[k].size());
    if (halo_rows) std::memcpy(halo_rows + o, p.halo0.rows[k].data(), p.halo0.rows[k].size() * sizeof(int32_t));
    o += static_cast<int64_t>(p.halo0.rows[k].size());
  }
  TS_API_END
}

ts_status ts_level2_setup_host(const ts_mesh* mesh, int32_t n_materials, const double* lambda, const double* mu,
                                const uint8_t* dof_mask, int32_t aggregate_target, int32_t* n2, int64_t* nnzb2) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && lambda && mu && n_materials >= 1, "level2 setup: null argument");
  const tsg::Mesh& m = mesh->m;
  const std::vector<uint8_t> gm = dof_mask ? std::vector<uint8_t>(dof_mask, dof_mask + 3 * size_t(m.n_nodes()))
                                           : m.dirichlet_mask();
  const std::vector<uint8_t> mask1(gm.begin(), gm.begin() + 3 * size_t(m.vertex_count));
  std::vector<double> le(m.n_elems()), me(m.n_elems());
  for (int32_t e = 0; e < m.n_elems(); ++e) {
    const int32_t k = m.material_id[e];
    TS_REQUIRE(k >= 0 && k < n_materials, "level2 setup: element references an undefined material");
    le[e] = lambda[k];
    me[e] = mu[k];
  }
  const tsg::Level2Host l2 = tsg::build_level2_host(m, le, me, mask1, aggregate_target);
  if (n2) *n2 = l2.n2;
  if (nnzb2) *nnzb2 = l2.row_ptr[l2.n2];
  TS_API_END
}

ts_status ts_dist_levels_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda, const double* mu,
                                const uint8_t* dof_mask, const int32_t* part, const ts_solver_config* cfg,
                                ts_comm* comm, ts_dist_levels** out) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && lambda && mu && part && cfg && comm && out, "dist levels: null argument");
  TS_REQUIRE(n_materials >= 1, "dist levels: need at least one material");
  TS_ABORT_ON_FAIL(comm->c, *out = tsg::dist_levels_create(mesh->m, n_materials, lambda, mu, dof_mask, part, *cfg,
                                                          comm->c.get()));
  TS_API_END
}

void ts_dist_levels_destroy(ts_dist_levels* lv) { tsg::dist_levels_destroy(lv); }

ts_status ts_dist_levels_sizes(const ts_dist_levels* lv, int32_t* n_local, int32_t* n_local_vertices, int32_t* n2) {
  TS_API_BEGIN
  TS_REQUIRE(lv, "dist levels: null handle");
  tsg::dist_levels_sizes(*lv, n_local, n_local_vertices, n2);
  TS_API_END
}

ts_status ts_dist_levels_info(const ts_dist_levels* lv, int32_t* n_elements, int64_t* halo_rows0,
                              int32_t* n_neighbours, double* setup_s) {
  TS_API_BEGIN
  TS_REQUIRE(lv && n_elements && halo_rows0 && n_neighbours && setup_s, "dist levels: null argument");
  tsg::dist_levels_info(*lv, n_elements, halo_rows0, n_neighbours, setup_s);
  TS_API_END
}

ts_status ts_dist_local_nodes(const ts_dist_levels* lv, int32_t* l2g) {
  TS_API_BEGIN
  TS_REQUIRE(lv && l2g, "dist levels: null argument");
  const auto& v = tsg::dist_local_nodes(*lv);
  std::memcpy(l2g, v.data(), v.size() * sizeof(int32_t));
  TS_API_END
}

ts_status ts_dist_solve(ts_dist_levels* lv, const double* f, const double* u0, double* u_out, int32_t n_local,
                        int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep) {
  TS_API_BEGIN
  TS_REQUIRE(lv && f && u0 && u_out && cfg && rep, "solve: null argument");
  TS_REQUIRE(size_t(n_local) == tsg::dist_local_nodes(*lv).size(), "solve: dimension mismatch");
  TS_ABORT_ON_FAIL(tsg::dist_levels_comm(*lv), tsg::dist_solve_host(*lv, f, u0, u_out, batch, *cfg, *rep));
  TS_API_END
}

ts_status ts_dist_solve_device(ts_dist_levels* lv, const double* f, const double* u0, double* u_out, int32_t n_local,
                               int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep, void* stream) {
  TS_API_BEGIN
  TS_REQUIRE(lv && f && u0 && u_out && cfg && rep, "solve: null argument");
  TS_REQUIRE(size_t(n_local) == tsg::dist_local_nodes(*lv).size(), "solve: dimension mismatch");
  TS_ABORT_ON_FAIL(tsg::dist_levels_comm(*lv),
                   tsg::dist_solve_device(*lv, f, u0, u_out, batch, *cfg, *rep, static_cast<cudaStream_t>(stream)));
  TS_API_END
}

ts_status ts_dist_ebe_apply(ts_dist_levels* lv, int32_t which, const void* u, void* f, int32_t batch, void* stream) {
  TS_API_BEGIN
  TS_REQUIRE(lv && u && f, "dist apply: null argument");
  TS_REQUIRE(batch >= 1, "dist apply: batch must be >= 1");
  TS_ABORT_ON_FAIL(tsg::dist_levels_comm(*lv),
                   tsg::dist_ebe_apply(*lv, which, u, f, batch, static_cast<cudaStream_t>(stream)));
  TS_API_END
}

ts_status ts_dist_ebe_create(const ts_mesh* mesh, int32_t order, int32_t n_materials, const double* lambda,
                             const double* mu, const uint8_t* dof_mask, const int32_t* part, int32_t prec,
                             ts_comm* comm, ts_dist_ebe** out) {
  TS_API_BEGIN
  TS_REQUIRE(mesh && lambda && mu && part && comm && out, "dist ebe: null argument");
  TS_REQUIRE(order == 1 || order == 2, "dist ebe: order must be 1 or 2");
  TS_REQUIRE(prec == 32 || prec == 64, "dist ebe: precision must be 32 or 64");
  TS_ABORT_ON_FAIL(comm->c, *out = tsg::dist_ebe_create(mesh->m, order, n_materials, lambda, mu, dof_mask, part,
                                                       prec, comm->c.get()));
  TS_API_END
}

void ts_dist_ebe_destroy(ts_dist_ebe* op) { tsg::dist_ebe_destroy(op); }

ts_status ts_dist_ebe_info(const ts_dist_ebe* op, int32_t* n_local, int32_t* n_elements, int64_t* halo_rows,
                           int32_t* n_neighbours) {
  TS_API_BEGIN
  TS_REQUIRE(op, "dist ebe: null handle");
  tsg::dist_ebe_info(*op, n_local, n_elements, halo_rows, n_neighbours);
  TS_API_END
}

ts_status ts_dist_ebe_local_nodes(const ts_dist_ebe* op, int32_t* l2g) {
  TS_API_BEGIN
  TS_REQUIRE(op && l2g, "dist ebe: null argument");
  const auto& v = tsg::dist_ebe_local_nodes(*op);
  std::memcpy(l2g, v.data(), v.size() * sizeof(int32_t));
  TS_API_END
}

ts_status ts_dist_ebe_op_apply(ts_dist_ebe* op, const void* u, void* f, int32_t batch, void* stream) {
  TS_API_BEGIN
  TS_REQUIRE(op && u && f, "dist ebe: null argument");
  TS_REQUIRE(batch >= 1, "dist ebe: batch must be >= 1");
  TS_ABORT_ON_FAIL(tsg::dist_ebe_comm(*op), tsg::dist_ebe_apply_op(*op, u, f, batch, static_cast<cudaStream_t>(stream)));
  TS_API_END
}

ts_status ts_dist_ebe_local_operator(ts_dist_ebe* op, ts_ebe** local) {
  TS_API_BEGIN
  TS_REQUIRE(op && local, "dist ebe: null argument");
  *local = tsg::dist_ebe_local(*op);
  TS_API_END
}

}  // extern "C"
