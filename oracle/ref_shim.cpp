// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Thin extern "C" shim over the UNMODIFIED reference headers, compiled in place
// from /root/reference/proj/include by oracle/Makefile into oracle/_ref/libtsref.so.
// Nothing here restates the algorithm: every numeric result comes from the
// reference's own code (tetsolve::EbeOperator, assemble_bcsr, build_solver_levels,
// solve, solve_pcge, ...). It exists so the pytest harness (and bench.py's
// cpu_baseline / --impl reference arm) can drive the reference through plain
// pointers. Only tests/, __graft_entry__.smoke() and bench.py may load it.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "tetsolve/adaptive_cg.hpp"
#include "tetsolve/box_mesh.hpp"
#include "tetsolve/fault.hpp"
#include "tetsolve/greens.hpp"
#include "tetsolve/mesh_io.hpp"
#include "tetsolve/model.hpp"
#include "tetsolve/solution_io.hpp"
#include "tetsolve/verification.hpp"

#include "../include/tsgpu.h"  // shared POD structs (ts_solver_config, ts_solve_report)

using namespace tetsolve;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_TRY try {
#define REF_CATCH                                                      \
  }                                                                    \
  catch (const ConvergenceError& e) { return fail(e, 4); }             \
  catch (const SolverError& e) { return fail(e, 2); }                  \
  catch (const ParseError& e) { return fail(e, 7); }                   \
  catch (const ValidationError& e) { return fail(e, 1); }              \
  catch (const std::exception& e) { return fail(e, 9); }               \
  return 0;

std::vector<Material> mats_of(int32_t n, const double* lam, const double* mu) {
  std::vector<Material> m(n);
  for (int32_t i = 0; i < n; ++i) {
    m[i].lambda = lam[i];
    m[i].mu = mu[i];
  }
  return m;
}

SolverConfig cfg_of(const ts_solver_config* c) {
  SolverConfig s;
  if (!c) return s;
  s.outer_tol = c->outer_tol;
  s.outer_max_iter = c->outer_max_iter;
  s.level0 = {c->level_tol[0], c->level_max_iter[0]};
  s.level1 = {c->level_tol[1], c->level_max_iter[1]};
  s.level2 = {c->level_tol[2], c->level_max_iter[2]};
  s.batch_size = c->batch_size;
  s.aggregate_target = c->aggregate_target;
  s.residual_history_stride = c->residual_history_stride;
  return s;
}

void report_out(const SolveReport& r, ts_solve_report* o) {
  if (!o) return;
  o->converged = r.converged;
  o->outer_iterations = r.outer_iterations;
  for (int i = 0; i < 3; ++i) {
    o->inner_iterations[i] = r.inner_iterations[i];
    o->time_inner_s[i] = r.time_inner_s[i];
  }
  o->time_setup_s = r.time_setup_s;
  o->time_outer_s = r.time_outer_s;
  o->time_total_s = r.time_total_s;
  o->batch_size = r.batch_size;
  o->method = r.method == "pcge" ? 1 : 0;
  o->inner_precision = r.inner_precision == "float64" ? 64 : 32;
  if (o->final_rel_residual)
    for (size_t b = 0; b < r.final_rel_residual.size(); ++b)
      o->final_rel_residual[b] = r.final_rel_residual[b];
  int32_t n = 0;
  for (const auto& [it, res] : r.residual_history) {
    if (n >= o->history_capacity) break;
    if (o->history_iter) o->history_iter[n] = it;
    if (o->history)
      for (size_t b = 0; b < res.size(); ++b) o->history[size_t(n) * res.size() + b] = res[b];
    ++n;
  }
  o->history_count = n;
}

template <typename T>
VectorBatch<T> batch_in(const void* p, int32_t nodes, int32_t batch) {
  VectorBatch<T> v(nodes, batch);
  if (p) std::memcpy(v.data.data(), p, v.data.size() * sizeof(T));
  return v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- meshes
void* ref_box_mesh(const double* ext, const int32_t* div, int32_t n_if, const double* ifs,
                   int32_t fixed) {
  try {
    BoxMeshSpec s;
    s.extents = {ext[0], ext[1], ext[2]};
    s.divisions = {div[0], div[1], div[2]};
    s.layer_interfaces.assign(ifs, ifs + n_if);
    s.fixed_boundary = fixed == 0   ? FixedBoundary::none
                       : fixed == 1 ? FixedBoundary::bottom_and_sides
                                    : FixedBoundary::all_clamped;
    return new Mesh(generate_box_mesh(s));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* ref_mesh_from_arrays(int32_t n_nodes, int32_t vertex_count, const double* coords,
                           int32_t n_elems, const int32_t* tets10, const int32_t* mat,
                           int32_t n_bc, const int32_t* bc_node, const int8_t* bc_axis) {
  auto* m = new Mesh;
  m->coords.resize(n_nodes);
  for (int32_t i = 0; i < n_nodes; ++i)
    m->coords[i] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
  m->vertex_count = vertex_count;
  m->tets10.resize(n_elems);
  m->tets4.resize(n_elems);
  m->material_id.assign(mat, mat + n_elems);
  for (int32_t e = 0; e < n_elems; ++e) {
    for (int a = 0; a < 10; ++a) m->tets10[e][a] = tets10[10 * size_t(e) + a];
    for (int a = 0; a < 4; ++a) m->tets4[e][a] = tets10[10 * size_t(e) + a];
  }
  for (int32_t i = 0; i < n_bc; ++i) m->dirichlet.push_back({bc_node[i], bc_axis[i]});
  rebuild_edge_map(*m);
  return m;
}

void ref_mesh_sizes(const void* h, int32_t* nn, int32_t* nv, int32_t* ne, int32_t* nbc) {
  const Mesh& m = *static_cast<const Mesh*>(h);
  *nn = m.node_count();
  *nv = m.vertex_count;
  *ne = m.element_count();
  *nbc = static_cast<int32_t>(m.dirichlet.size());
}

void ref_mesh_export(const void* h, double* coords, int32_t* tets10, int32_t* mat,
                     int32_t* bc_node, int8_t* bc_axis) {
  const Mesh& m = *static_cast<const Mesh*>(h);
  if (coords)
    for (int32_t i = 0; i < m.node_count(); ++i)
      for (int c = 0; c < 3; ++c) coords[3 * size_t(i) + c] = m.coords[i][c];
  if (tets10)
    for (int32_t e = 0; e < m.element_count(); ++e)
      for (int a = 0; a < 10; ++a) tets10[10 * size_t(e) + a] = m.tets10[e][a];
  if (mat) std::copy(m.material_id.begin(), m.material_id.end(), mat);
  for (size_t i = 0; i < m.dirichlet.size(); ++i) {
    if (bc_node) bc_node[i] = m.dirichlet[i].node;
    if (bc_axis) bc_axis[i] = m.dirichlet[i].axis;
  }
}

void ref_mesh_mask(const void* h, uint8_t* mask) {
  const auto v = dirichlet_mask(*static_cast<const Mesh*>(h));
  std::copy(v.begin(), v.end(), mask);
}

void ref_mesh_destroy(void* h) { delete static_cast<Mesh*>(h); }

int ref_material_from_wavespeeds(double vp, double vs, double rho, double* lam, double* mu) {
  REF_TRY
  const Material m = material_from_wavespeeds(vp, vs, rho);
  *lam = m.lambda;
  *mu = m.mu;
  REF_CATCH
}

// -------------------------------------------------------------- element
int ref_element_matrix(int32_t order, const double* v12, double lam, double mu, double* k) {
  REF_TRY
  Vec3 v[4];
  for (int a = 0; a < 4; ++a) v[a] = {v12[3 * a], v12[3 * a + 1], v12[3 * a + 2]};
  if (order == 1)
    detail::tet4_stiffness_kernel(v, lam, mu, k);
  else
    detail::tet10_stiffness_kernel(v, lam, mu, k);
  REF_CATCH
}

// ------------------------------------------------------------ operators
// mask == nullptr => unconstrained; else 3*n_nodes(order) bytes.
int ref_ebe_apply(const void* mh, int32_t order, int32_t n_mat, const double* lam,
                  const double* mu, const uint8_t* mask, int32_t prec, int32_t workers,
                  const void* u, void* f, int32_t batch) {
  REF_TRY
  const Mesh& m = *static_cast<const Mesh*>(mh);
  const int32_t nn = order == 1 ? m.vertex_count : m.node_count();
  std::vector<uint8_t> mk;
  if (mask) mk.assign(mask, mask + 3 * size_t(nn));
  if (prec == 64) {
    EbeOperator<double> op(m, order, mats_of(n_mat, lam, mu), mk, workers);
    const auto ub = batch_in<double>(u, nn, batch);
    VectorBatch64 fb;
    op.apply(ub, fb);
    std::memcpy(f, fb.data.data(), fb.data.size() * sizeof(double));
  } else {
    EbeOperator<float> op(m, order, mats_of(n_mat, lam, mu), mk, workers);
    const auto ub = batch_in<float>(u, nn, batch);
    VectorBatch32 fb;
    op.apply(ub, fb);
    std::memcpy(f, fb.data.data(), fb.data.size() * sizeof(float));
  }
  REF_CATCH
}

// Time EbeOperator<T>::apply (1 warm-up + reps timed applies) on inputs
// DeterministicRng(seed).sym() (verification.hpp:29-31); returns seconds/apply.
int ref_time_ebe_apply(const void* mh, int32_t order, int32_t n_mat, const double* lam,
                       const double* mu, int32_t use_mask, int32_t prec, int32_t workers,
                       int32_t batch, int32_t reps, uint64_t seed, double* sec_per_apply,
                       double* checksum) {
  REF_TRY
  const Mesh& m = *static_cast<const Mesh*>(mh);
  std::vector<uint8_t> mk;
  if (use_mask) {
    mk = dirichlet_mask(m);
    if (order == 1) mk.resize(3 * size_t(m.vertex_count));
  }
  auto run = [&](auto tag) {
    using T = decltype(tag);
    EbeOperator<T> op(m, order, mats_of(n_mat, lam, mu), mk, workers);
    DeterministicRng rng(seed);
    VectorBatch<T> u(op.n_nodes(), batch), f;
    for (auto& x : u.data) x = static_cast<T>(rng.sym());
    op.apply(u, f);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) op.apply(u, f);
    const auto t1 = std::chrono::steady_clock::now();
    *sec_per_apply = std::chrono::duration<double>(t1 - t0).count() / std::max(reps, 1);
    double s = 0.0;
    for (T x : f.data) s += double(x);
    *checksum = s;
  };
  if (prec == 64) run(double{});
  else run(float{});
  REF_CATCH
}

// assemble_bcsr(EbeOperator<T>) (ebe_operator.hpp:230-284); blocks exported as double.
void* ref_assemble_bcsr(const void* mh, int32_t order, int32_t n_mat, const double* lam,
                        const double* mu, const uint8_t* mask, int32_t prec) {
  try {
    const Mesh& m = *static_cast<const Mesh*>(mh);
    const int32_t nn = order == 1 ? m.vertex_count : m.node_count();
    std::vector<uint8_t> mk;
    if (mask) mk.assign(mask, mask + 3 * size_t(nn));
    auto* out = new BlockCsrMatrix<double>;
    if (prec == 64) {
      EbeOperator<double> op(m, order, mats_of(n_mat, lam, mu), mk, 1);
      *out = assemble_bcsr(op);
    } else {
      EbeOperator<float> op(m, order, mats_of(n_mat, lam, mu), mk, 1);
      *out = cast_bcsr<double>(assemble_bcsr(op));
    }
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_bcsr_sizes(const void* h, int32_t* nrows, int64_t* nnzb) {
  const auto& a = *static_cast<const BlockCsrMatrix<double>*>(h);
  *nrows = a.n_block_rows;
  *nnzb = a.n_blocks();
}

void ref_bcsr_export(const void* h, int32_t* row_ptr, int32_t* col_idx, double* blocks) {
  const auto& a = *static_cast<const BlockCsrMatrix<double>*>(h);
  std::copy(a.row_ptr.begin(), a.row_ptr.end(), row_ptr);
  std::copy(a.col_idx.begin(), a.col_idx.end(), col_idx);
  for (size_t e = 0; e < a.blocks.size(); ++e)
    for (int q = 0; q < 9; ++q) blocks[9 * e + q] = a.blocks[e][q];
}

void ref_bcsr_destroy(void* h) { delete static_cast<BlockCsrMatrix<double>*>(h); }

// BlockCsrMatrix<T>::apply (block_csr.hpp:33-69) on raw arrays; blocks given in T.
int ref_bcsr_apply(int32_t nrows, const int32_t* row_ptr, const int32_t* col_idx,
                   const void* blocks, int32_t prec, const void* u, void* f, int32_t batch) {
  REF_TRY
  auto run = [&](auto tag) {
    using T = decltype(tag);
    BlockCsrMatrix<T> a;
    a.n_block_rows = nrows;
    a.row_ptr.assign(row_ptr, row_ptr + nrows + 1);
    a.col_idx.assign(col_idx, col_idx + row_ptr[nrows]);
    a.blocks.resize(a.col_idx.size());
    std::memcpy(a.blocks.data(), blocks, a.blocks.size() * 9 * sizeof(T));
    const auto ub = batch_in<T>(u, nrows, batch);
    VectorBatch<T> fb;
    a.apply(ub, fb);
    std::memcpy(f, fb.data.data(), fb.data.size() * sizeof(T));
  };
  if (prec == 64) run(double{});
  else run(float{});
  REF_CATCH
}

// extract_block_jacobi(EbeOperator<T>) (ebe_operator.hpp:288-313); inv in T.
int ref_ebe_block_jacobi(const void* mh, int32_t order, int32_t n_mat, const double* lam,
                         const double* mu, const uint8_t* mask, int32_t prec, void* inv) {
  REF_TRY
  const Mesh& m = *static_cast<const Mesh*>(mh);
  const int32_t nn = order == 1 ? m.vertex_count : m.node_count();
  std::vector<uint8_t> mk;
  if (mask) mk.assign(mask, mask + 3 * size_t(nn));
  auto run = [&](auto tag) {
    using T = decltype(tag);
    EbeOperator<T> op(m, order, mats_of(n_mat, lam, mu), mk, 1);
    const BlockJacobi<T> bj = extract_block_jacobi(op);
    std::memcpy(inv, bj.inv_blocks.data(), bj.inv_blocks.size() * 9 * sizeof(T));
  };
  if (prec == 64) run(double{});
  else run(float{});
  REF_CATCH
}

// BlockJacobi<T>::apply (block_jacobi.hpp:22-38)
int ref_bj_apply(int32_t n, const void* inv, int32_t prec, const void* r, void* z, int32_t batch) {
  REF_TRY
  auto run = [&](auto tag) {
    using T = decltype(tag);
    BlockJacobi<T> bj;
    bj.inv_blocks.resize(n);
    std::memcpy(bj.inv_blocks.data(), inv, size_t(n) * 9 * sizeof(T));
    const auto rb = batch_in<T>(r, n, batch);
    VectorBatch<T> zb;
    bj.apply(rb, zb);
    std::memcpy(z, zb.data.data(), zb.data.size() * sizeof(T));
  };
  if (prec == 64) run(double{});
  else run(float{});
  REF_CATCH
}

// Geometric prolongation P1 -> P2 (prolongation.hpp:67-98) apply / restrict (fp32).
int ref_geo_prolong(const void* mh, int32_t transpose, const float* in, float* out, int32_t batch) {
  REF_TRY
  const Mesh& m = *static_cast<const Mesh*>(mh);
  const Prolongation p = build_geometric_prolongation(m);
  if (!transpose) {
    const auto c = batch_in<float>(in, p.n_coarse_nodes, batch);
    VectorBatch32 fo;
    p.apply(c, fo);
    std::memcpy(out, fo.data.data(), fo.data.size() * sizeof(float));
  } else {
    const auto fi = batch_in<float>(in, p.n_fine_nodes, batch);
    VectorBatch32 co;
    p.restrict_to_coarse(fi, co);
    std::memcpy(out, co.data.data(), co.data.size() * sizeof(float));
  }
  REF_CATCH
}

// inner_pcg (pcg.hpp:52-124) on EbeOperator<float> with its own block Jacobi.
int ref_inner_pcg_ebe(const void* mh, int32_t order, int32_t n_mat, const double* lam,
                      const double* mu, const uint8_t* mask, const float* r, float* u,
                      int32_t batch, double tol, int32_t max_iter, int32_t* iters,
                      int32_t* converged) {
  REF_TRY
  const Mesh& m = *static_cast<const Mesh*>(mh);
  const int32_t nn = order == 1 ? m.vertex_count : m.node_count();
  std::vector<uint8_t> mk;
  if (mask) mk.assign(mask, mask + 3 * size_t(nn));
  EbeOperator<float> op(m, order, mats_of(n_mat, lam, mu), mk, 1);
  const BlockJacobi<float> bj = extract_block_jacobi(op);
  const auto rb = batch_in<float>(r, nn, batch);
  auto ub = batch_in<float>(u, nn, batch);
  PcgWork<float> w;
  const InnerStats st = inner_pcg(op, bj, rb, ub, tol, max_iter, w);
  std::memcpy(u, ub.data.data(), ub.data.size() * sizeof(float));
  *iters = st.iterations;
  *converged = st.converged;
  REF_CATCH
}

// ------------------------------------------------------------ level set
void* ref_levels_create(const void* mh, int32_t n_mat, const double* lam, const double* mu,
                        const ts_solver_config* cfg, int32_t workers, double* setup_s) {
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const Mesh& m = *static_cast<const Mesh*>(mh);
    auto* lv = new SolverLevels(
        build_solver_levels(m, mats_of(n_mat, lam, mu), dirichlet_mask(m), cfg_of(cfg), workers));
    if (setup_s)
      *setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return lv;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_levels_sizes(const void* h, int32_t* n0, int32_t* n1, int32_t* n2, int64_t* nnzb2) {
  const auto& lv = *static_cast<const SolverLevels*>(h);
  *n0 = lv.level0.n_nodes();
  *n1 = lv.level1.n_nodes();
  *n2 = lv.level2.n_block_rows;
  *nnzb2 = lv.level2.n_blocks();
}

void ref_levels_export(const void* h, int32_t* agg, int32_t* row_ptr2, int32_t* col_idx2,
                       float* blocks2, uint8_t* mask2, float* m0, float* m1, float* m2) {
  const auto& lv = *static_cast<const SolverLevels*>(h);
  if (agg) std::copy(lv.aggregation.agg_of_node.begin(), lv.aggregation.agg_of_node.end(), agg);
  if (row_ptr2) std::copy(lv.level2.row_ptr.begin(), lv.level2.row_ptr.end(), row_ptr2);
  if (col_idx2) std::copy(lv.level2.col_idx.begin(), lv.level2.col_idx.end(), col_idx2);
  if (blocks2) std::memcpy(blocks2, lv.level2.blocks.data(), lv.level2.blocks.size() * 36);
  if (mask2) std::copy(lv.mask2.begin(), lv.mask2.end(), mask2);
  if (m0) std::memcpy(m0, lv.m0.inv_blocks.data(), lv.m0.inv_blocks.size() * 36);
  if (m1) std::memcpy(m1, lv.m1.inv_blocks.data(), lv.m1.inv_blocks.size() * 36);
  if (m2) std::memcpy(m2, lv.m2.inv_blocks.data(), lv.m2.inv_blocks.size() * 36);
}

void ref_levels_destroy(void* h) { delete static_cast<SolverLevels*>(h); }

// the level set's own 64-bit outer operator applied to u (manufactured RHS)
int ref_levels_outer_apply(const void* h, const double* u, double* f, int32_t batch) {
  REF_TRY
  const auto& lv = *static_cast<const SolverLevels*>(h);
  const auto ub = batch_in<double>(u, lv.outer.n_nodes(), batch);
  VectorBatch64 fb;
  lv.outer.apply(ub, fb);
  std::memcpy(f, fb.data.data(), fb.data.size() * sizeof(double));
  REF_CATCH
}

int ref_solve(const void* h, const double* f, const double* u0, double* u_out, int32_t batch,
              const ts_solver_config* cfg, ts_solve_report* rep) {
  const auto& lv = *static_cast<const SolverLevels*>(h);
  const int32_t nn = lv.outer.n_nodes();
  try {
    const auto fb = batch_in<double>(f, nn, batch);
    const auto u0b = batch_in<double>(u0, nn, batch);
    auto [u, r] = solve(lv, fb, u0b, cfg_of(cfg));
    std::memcpy(u_out, u.data.data(), u.data.size() * sizeof(double));
    report_out(r, rep);
  } catch (const ConvergenceError& e) {
    report_out(e.report, rep);
    return fail(e, 4);
  } catch (const SolverError& e) {
    return fail(e, 2);
  } catch (const ValidationError& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
  return 0;
}

int ref_solve_pcge(const void* h, const double* f, const double* u0, double* u_out,
                   int32_t batch, double tol, int32_t max_iter, ts_solve_report* rep) {
  const auto& lv = *static_cast<const SolverLevels*>(h);
  const int32_t nn = lv.outer.n_nodes();
  try {
    const auto fb = batch_in<double>(f, nn, batch);
    const auto u0b = batch_in<double>(u0, nn, batch);
    auto [u, r] = solve_pcge(lv.outer, fb, u0b, tol, max_iter);
    std::memcpy(u_out, u.data.data(), u.data.size() * sizeof(double));
    report_out(r, rep);
  } catch (const ConvergenceError& e) {
    report_out(e.report, rep);
    return fail(e, 4);
  } catch (const SolverError& e) {
    return fail(e, 2);
  } catch (const ValidationError& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
  return 0;
}

// DeterministicRng stream (verification.hpp:14-19) for golden inputs.
void ref_rng_sym(uint64_t seed, int64_t n, double* out) {
  DeterministicRng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.sym();
}

int ref_hw_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// ---- Green's-function sweep (fault.hpp / model.hpp / greens.hpp), for parity tests
int ref_fault_plane_faces(const void* mh, int32_t axis, double coord, const double* lo, const double* hi,
                          int32_t* n_faces, int32_t* faces) {
  REF_TRY
  const auto f = find_plane_fault_faces(*static_cast<const Mesh*>(mh), axis, coord, {lo[0], lo[1], lo[2]},
                                        {hi[0], hi[1], hi[2]});
  if (faces)
    for (size_t i = 0; i < f.size() && int32_t(i) < *n_faces; ++i)
      for (int k = 0; k < 3; ++k) faces[3 * i + k] = f[i][k];
  *n_faces = static_cast<int32_t>(f.size());
  REF_CATCH
}

namespace {
std::vector<std::array<int32_t, 3>> tris_of(const int32_t* faces, int32_t n) {
  std::vector<std::array<int32_t, 3>> t(n);
  for (int32_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) t[i][k] = faces[3 * i + k];
  return t;
}
std::vector<UnitSlip> slips_of(const FaultedModel& fm, int32_t n, const double* c, const int32_t* d, const double* r) {
  std::vector<UnitSlip> s;
  for (int32_t j = 0; j < n; ++j)
    s.push_back(unit_slip_basis(fm.patch, fm.base.mesh, {c[3 * j], c[3 * j + 1], c[3 * j + 2]},
                                d[j] == 0 ? SlipDirection::dip : SlipDirection::strike, r[j]));
  return s;
}
}  // namespace

int ref_slip_to_rhs(const void* mh, int32_t n_mat, const double* lam, const double* mu, const int32_t* faces,
                    int32_t n_faces, int32_t n_slips, const double* centers, const int32_t* dirs, const double* radii,
                    double* f_out, int32_t* split_info /*[2]: split nodes, split mesh nodes*/) {
  REF_TRY
  const FaultedModel fm = build_faulted_model(*static_cast<const Mesh*>(mh), mats_of(n_mat, lam, mu),
                                              tris_of(faces, n_faces), SolverConfig{});
  const auto slips = slips_of(fm, n_slips, centers, dirs, radii);
  const int32_t N = fm.base.mesh.node_count();
  for (int32_t j = 0; j < n_slips; ++j) {
    const VectorBatch64 col = slip_to_rhs(fm, slips[j]);
    for (int64_t d = 0; d < 3 * int64_t(N); ++d) f_out[d * n_slips + j] = col.at(d, 0);
  }
  if (split_info) {
    split_info[0] = static_cast<int32_t>(fm.patch.split_nodes.size());
    split_info[1] = fm.split_mesh.node_count();
  }
  REF_CATCH
}

int ref_greens_bank(const void* mh, int32_t n_mat, const double* lam, const double* mu, const int32_t* faces,
                    int32_t n_faces, int32_t n_slips, const double* centers, const int32_t* dirs, const double* radii,
                    int32_t n_obs, const double* points, const int32_t* axes, const ts_solver_config* cfg,
                    double* bank, int32_t* solver_calls, int64_t* outer_iterations) {
  REF_TRY
  const SolverConfig c = cfg_of(cfg);
  const FaultedModel fm = build_faulted_model(*static_cast<const Mesh*>(mh), mats_of(n_mat, lam, mu),
                                              tris_of(faces, n_faces), c);
  const auto slips = slips_of(fm, n_slips, centers, dirs, radii);
  std::vector<ObservationComponent> obs(n_obs);
  for (int32_t r = 0; r < n_obs; ++r) {
    obs[r].point = {points[3 * r], points[3 * r + 1], points[3 * r + 2]};
    obs[r].axis = axes[r];
  }
  auto [b, rep] = compute_greens_bank(fm, slips, obs, c);
  std::memcpy(bank, b.values.data(), b.values.size() * sizeof(double));
  *solver_calls = rep.solver_calls;
  *outer_iterations = rep.outer_iterations;
  REF_CATCH
}

// ------------------------------------------------------------ file formats
// write_mesh / read_mesh / write_dirichlet / read_dirichlet (mesh_io.hpp),
// write_solution / read_solution (solution_io.hpp)
int ref_write_mesh(const void* mh, const char* path) {
  REF_TRY
  write_mesh(*static_cast<const Mesh*>(mh), path);
  REF_CATCH
}

int ref_read_mesh(const char* path, void** out) {
  REF_TRY
  *out = new Mesh(read_mesh(path));
  REF_CATCH
}

int ref_write_dirichlet(const void* mh, const char* path) {
  REF_TRY
  write_dirichlet(*static_cast<const Mesh*>(mh), path);
  REF_CATCH
}

int ref_read_dirichlet(void* mh, const char* path) {
  REF_TRY
  read_dirichlet(*static_cast<Mesh*>(mh), path);
  REF_CATCH
}

int ref_write_solution(const char* path, const double* u, int32_t nodes, int32_t batch) {
  REF_TRY
  VectorBatch64 v(nodes, batch);
  std::memcpy(v.data.data(), u, v.data.size() * sizeof(double));
  write_solution(v, path);
  REF_CATCH
}

// out == nullptr: dimensions only
int ref_read_solution(const char* path, int32_t* nodes, int32_t* batch, double* out) {
  REF_TRY
  const VectorBatch64 v = read_solution(path);
  *nodes = v.n_nodes;
  *batch = v.batch;
  if (out) std::memcpy(out, v.data.data(), v.data.size() * sizeof(double));
  REF_CATCH
}

// write_fault_faces / read_fault_faces (fault.hpp), read_observations / write_greens_bank /
// read_greens_bank (greens.hpp)
int ref_write_fault_faces(const char* path, const int32_t* faces, int32_t n) {
  REF_TRY
  std::vector<std::array<int32_t, 3>> f(n);
  for (int32_t i = 0; i < n; ++i) f[i] = {faces[3 * i], faces[3 * i + 1], faces[3 * i + 2]};
  write_fault_faces(f, path);
  REF_CATCH
}

int ref_read_fault_faces(const char* path, int32_t* n, int32_t* faces) {
  REF_TRY
  const auto f = read_fault_faces(path);
  *n = static_cast<int32_t>(f.size());
  if (faces)
    for (size_t i = 0; i < f.size(); ++i)
      for (int k = 0; k < 3; ++k) faces[3 * i + k] = f[i][k];
  REF_CATCH
}

int ref_read_observations(const char* path, int32_t* n, double* points, int32_t* axes) {
  REF_TRY
  const auto o = read_observations(path);
  *n = static_cast<int32_t>(o.size());
  for (size_t i = 0; i < o.size(); ++i) {
    if (points)
      for (int c = 0; c < 3; ++c) points[3 * i + c] = o[i].point[c];
    if (axes) axes[i] = o[i].axis;
  }
  REF_CATCH
}

int ref_write_greens_bank(const char* path, int32_t rows, int32_t cols, const double* pts, const int32_t* axes,
                          const double* centers, const int32_t* dirs, const double* radii, const double* values) {
  REF_TRY
  GreensBank b;
  b.rows = rows;
  b.cols = cols;
  b.values.assign(values, values + size_t(rows) * cols);
  for (int32_t r = 0; r < rows; ++r) b.obs.push_back({{pts[3 * r], pts[3 * r + 1], pts[3 * r + 2]}, axes[r]});
  for (int32_t c = 0; c < cols; ++c)
    b.columns.push_back({{centers[3 * c], centers[3 * c + 1], centers[3 * c + 2]},
                         dirs[c] == 0 ? SlipDirection::dip : SlipDirection::strike, radii[c]});
  write_greens_bank(b, path);
  REF_CATCH
}

int ref_read_greens_bank(const char* path, int32_t* rows, int32_t* cols, double* pts, int32_t* axes, double* centers,
                         int32_t* dirs, double* radii, double* values) {
  REF_TRY
  const GreensBank b = read_greens_bank(path);
  *rows = b.rows;
  *cols = b.cols;
  if (values) std::copy(b.values.begin(), b.values.end(), values);
  for (int32_t r = 0; r < b.rows; ++r) {
    if (pts)
      for (int c = 0; c < 3; ++c) pts[3 * r + c] = b.obs[r].point[c];
    if (axes) axes[r] = b.obs[r].axis;
  }
  for (int32_t c = 0; c < b.cols; ++c) {
    if (centers)
      for (int k = 0; k < 3; ++k) centers[3 * c + k] = b.columns[c].center[k];
    if (dirs) dirs[c] = b.columns[c].direction == SlipDirection::dip ? 0 : 1;
    if (radii) radii[c] = b.columns[c].radius;
  }
  REF_CATCH
}

// reconstruct_split_solution (fault.hpp:392-411) of each slip's column of u_base
int ref_reconstruct_split(const void* mh, int32_t n_mat, const double* lam, const double* mu, const int32_t* faces,
                          int32_t n_faces, int32_t n_slips, const double* centers, const int32_t* dirs,
                          const double* radii, const double* u_base, double* u_split) {
  REF_TRY
  const FaultedModel fm = build_faulted_model(*static_cast<const Mesh*>(mh), mats_of(n_mat, lam, mu),
                                              tris_of(faces, n_faces), SolverConfig{});
  const auto slips = slips_of(fm, n_slips, centers, dirs, radii);
  const int32_t N = fm.base.mesh.node_count(), NS = fm.split_mesh.node_count();
  for (int32_t j = 0; j < n_slips; ++j) {
    VectorBatch64 ub(N, 1);
    for (int64_t d = 0; d < 3 * int64_t(N); ++d) ub.at(d, 0) = u_base[d * n_slips + j];
    const VectorBatch64 us = reconstruct_split_solution(fm.patch, slip_vectors(fm.patch, slips[j]), ub, NS);
    for (int64_t d = 0; d < 3 * int64_t(NS); ++d) u_split[d * n_slips + j] = us.at(d, 0);
  }
  REF_CATCH
}

}  // extern "C"
