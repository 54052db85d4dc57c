// solver.cu — the device-resident solve path: inner PCG (pcg.hpp:52-124),
// the 3-level mixed-precision multigrid preconditioner (adaptive_cg.hpp:80-120),
// the fp64 flexible outer CG (adaptive_cg.hpp:126-233), solve / solve_pcge
// (adaptive_cg.hpp:242-279) and the level-set construction
// (build_solver_levels, adaptive_cg.hpp:39-67).
//
// All vectors live in HBM for the whole solve; the host only sequences
// kernels and reads one 24-byte status record per iteration (the reference's
// convergence test is a host-side max over columns, pcg.hpp:71,116-117).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>

#include "blas.h"
#include "ebe.h"
#include "setup.h"
#include "solver_core.h"

using tsg::ColScalars;
using tsg::DevBuf;

struct LevelVecs {
  int32_t batch = 0;
  DevBuf<double> r, q, z, p, scratch, f, u;  // outer (fp64); f/u used by the host-buffer entry
  DevBuf<float> r0, u0, e0, p0, q0;          // level 0 (N nodes)
  DevBuf<float> r1, u1, e1, p1, q1;          // level 1 (V nodes)
  DevBuf<float> r2, u2, e2, p2, q2;          // level 2 (n2 nodes)
};

struct ts_levels {
  int32_t n0 = 0, n1 = 0, n2 = 0;
  std::unique_ptr<ts_ebe> outer, l0, l1;
  DevBuf<int32_t> l2_row_ptr, l2_col_idx;
  DevBuf<float> l2_blocks;
  // level 1 as an assembled BCSR (float-rounded assembly of the fp32 tet4 operator):
  // tet4's ~21 elements per vertex make the EBE scatter L2-atomic bound
  bool l1_assembled = false;
  DevBuf<int32_t> l1_row_ptr, l1_col_idx;
  DevBuf<float> l1_blocks;
  DevBuf<int32_t> p1_ends, p1t_ptr, p1t_idx, agg, p2t_ptr, p2t_idx;
  DevBuf<float> m0, m1, m2;
  DevBuf<uint8_t> mask0, mask1, mask2;
  std::vector<int32_t> h_agg, h_seeds, h_rp2, h_ci2;
  std::vector<float> h_bl2, h_m2;
  std::vector<uint8_t> h_mask2;
  double setup_s = 0.0;
  LevelVecs v;
  ColScalars cs;
  tsg::Workspace ws;
  std::mutex mu;
  DevBuf<double> host_f, host_u;  // staging of the host-buffer entry, kept across calls (no per-call cudaMalloc)
};

namespace tsg {
namespace {
using namespace core;

void ensure_vecs(ts_levels& lv, int32_t B) {
  LevelVecs& v = lv.v;
  if (v.batch == B) return;
  const size_t l0 = 3 * size_t(lv.n0) * B, l1 = 3 * size_t(lv.n1) * B, l2 = 3 * size_t(lv.n2) * B;
  for (auto* b : {&v.r, &v.q, &v.z, &v.p, &v.scratch}) b->alloc(l0);
  for (auto* b : {&v.r0, &v.u0, &v.e0, &v.p0, &v.q0}) b->alloc(l0);
  for (auto* b : {&v.r1, &v.u1, &v.e1, &v.p1, &v.q1}) b->alloc(l1);
  for (auto* b : {&v.r2, &v.u2, &v.e2, &v.p2, &v.q2}) b->alloc(l2);
  v.f.release();
  v.u.release();
  v.batch = B;
  lv.cs.ensure(B);
  lv.ws.ensure(B);
}

// apply_multigrid_preconditioner (adaptive_cg.hpp:80-120)
void mg_precond(ts_levels& lv, const ts_solver_config& cfg, const double* r, double* z, int32_t B,
                ts_solve_report& rep, cudaStream_t s) {
  NvtxRange nv("mg preconditioner");
  LevelVecs& v = lv.v;
  const int64_t len0 = 3 * int64_t(lv.n0) * B;
  cast_d2f(r, v.r0.get(), len0, s);
  bj_apply<float>(lv.m0.get(), v.r0.get(), v.u0.get(), lv.n0, B, s);
  p1_restrict(v.r0.get(), v.r1.get(), lv.p1t_ptr.get(), lv.p1t_idx.get(), lv.n1, lv.mask1.get(), B, s);
  p1_restrict(v.u0.get(), v.u1.get(), lv.p1t_ptr.get(), lv.p1t_idx.get(), lv.n1, lv.mask1.get(), B, s);
  p2_restrict(v.r1.get(), v.r2.get(), lv.p2t_ptr.get(), lv.p2t_idx.get(), lv.n2, lv.mask2.get(), B, s);
  p2_restrict(v.u1.get(), v.u2.get(), lv.p2t_ptr.get(), lv.p2t_idx.get(), lv.n2, lv.mask2.get(), B, s);
  const auto t0 = clk::now();
  auto a2 = [&](const float* x, float* y, bool) {
    bcsr_apply_f32(lv.l2_row_ptr.get(), lv.l2_col_idx.get(), lv.l2_blocks.get(), lv.n2, x, y, B, s,
                   static_cast<int64_t>(lv.l2_col_idx.size()));
  };
  const std::function<int(const float*, float*)> a2_dots = [&](const float* x, float* y) {
    return bcsr_apply_f32_gamma(lv.l2_row_ptr.get(), lv.l2_col_idx.get(), lv.l2_blocks.get(), lv.n2, x, y, B, s,
                                static_cast<int64_t>(lv.l2_col_idx.size()), lv.ws)
               ? 1 : 0;
  };
  InnerStats s2;
  {
    NvtxRange nl("inner pcg level 2");
    s2 = inner_pcg<float>(a2, lv.m2.get(), v.r2.get(), v.u2.get(), lv.n2, B, cfg.level_tol[2], cfg.level_max_iter[2],
                          v.e2.get(), v.p2.get(), v.q2.get(), lv.cs, lv.ws, s, false, nullptr, &a2_dots);
  }
  const auto t1 = clk::now();
  p2_apply(v.u2.get(), v.u1.get(), lv.agg.get(), lv.n1, lv.mask1.get(), B, s);
  auto a1 = [&](const float* x, float* y, bool init) {
    if (lv.l1_assembled)
      bcsr_rows_f32(lv.l1_row_ptr.get(), lv.l1_col_idx.get(), lv.l1_blocks.get(), lv.n1, x, y, B, s, nullptr,
                    static_cast<int64_t>(lv.l1_col_idx.size()));
    else
      ebe_apply_part(*lv.l1, x, y, B, s, -1, init);
  };
  const std::function<int(const float*, float*)> a1_dots = [&](const float* x, float* y) {
    return lv.l1_assembled && bcsr_rows_f32_gamma(lv.l1_row_ptr.get(), lv.l1_col_idx.get(), lv.l1_blocks.get(),
                                                   lv.n1, x, y, B, s, static_cast<int64_t>(lv.l1_col_idx.size()),
                                                   lv.ws)
               ? 1 : 0;
  };
  InnerStats s1;
  {
    NvtxRange nl("inner pcg level 1");
    s1 = inner_pcg<float>(a1, lv.m1.get(), v.r1.get(), v.u1.get(), lv.n1, B, cfg.level_tol[1], cfg.level_max_iter[1],
                          v.e1.get(), v.p1.get(), v.q1.get(), lv.cs, lv.ws, s, !lv.l1_assembled, lv.mask1.get(),
                          &a1_dots);
  }
  const auto t2 = clk::now();
  p1_apply(v.u1.get(), v.u0.get(), lv.p1_ends.get(), lv.n1, lv.n0, lv.mask0.get(), B, s);
  auto a0 = [&](const float* x, float* y, bool init) { ebe_apply_part(*lv.l0, x, y, B, s, -1, init); };
  // q's start is written by the direction pass (fuse_init), so the dots product adds onto it
  const std::function<int(const float*, float*)> a0_dots = [&](const float* x, float* y) {
    if (lv.ws.comm || lv.ws.owned) return 0;
    lv.ws.ensure(B);
    const int nb = ebe_pair_apply_dots(*lv.l0, x, y, B, s, lv.ws.partial.get());
    if (nb < 0) return 0;
    lv.ws.nblk = nb;
    return 2;
  };
  InnerStats s0;
  {
    NvtxRange nl("inner pcg level 0");
    s0 = inner_pcg<float>(a0, lv.m0.get(), v.r0.get(), v.u0.get(), lv.n0, B, cfg.level_tol[0], cfg.level_max_iter[0],
                          v.e0.get(), v.p0.get(), v.q0.get(), lv.cs, lv.ws, s, true, lv.mask0.get(), &a0_dots);
  }
  const auto t3 = clk::now();
  rep.inner_iterations[2] += s2.iterations;
  rep.inner_iterations[1] += s1.iterations;
  rep.inner_iterations[0] += s0.iterations;
  rep.time_inner_s[2] += secs(t0, t1);
  rep.time_inner_s[1] += secs(t1, t2);
  rep.time_inner_s[0] += secs(t2, t3);
  cast_f2d(v.u0.get(), z, len0, s);
}

void check_cfg(const ts_solver_config* c) {
  const ts_status rc = ts_config_validate(c);
  if (rc != TS_OK) fail(rc, ts_last_error());
}

// solve (adaptive_cg.hpp:242-263) on device buffers
void solve_device(ts_levels& lv, const double* f, const double* u0, double* u, int32_t B, const ts_solver_config& cfg,
                  ts_solve_report& rep, cudaStream_t s) {
  NvtxRange nv("tetsolve solve");
  check_cfg(&cfg);
  if (B < 1 || B > kRedThreads) validation("solve: batch must be in [1, 256]");
  ensure_vecs(lv, B);
  dot2<double>(f, f, nullptr, nullptr, 3 * int64_t(lv.n0), B, lv.cs[ColScalars::FN2], lv.ws, s);
  std::vector<double> fn2(B);
  TS_CUDA(cudaMemcpyAsync(fn2.data(), lv.cs[ColScalars::FN2], B * sizeof(double), cudaMemcpyDeviceToHost, s));
  TS_CUDA(cudaStreamSynchronize(s));
  bool any = false;
  for (double x : fn2) any |= x != 0.0;
  if (!any) validation("solve: right-hand side has no nonzero column");
  report_reset(rep, 0, 32);
  rep.time_setup_s = lv.setup_s;
  if (u != u0)
    TS_CUDA(cudaMemcpyAsync(u, u0, 3 * size_t(lv.n0) * B * sizeof(double), cudaMemcpyDeviceToDevice, s));
  auto precond = [&](const double* r, double* z) { mg_precond(lv, cfg, r, z, B, rep, s); };
  auto kop = [&](const double* x, double* y) { ebe_apply(*lv.outer, x, y, B, s); };
  run_outer_cg(kop, lv.n0, f, u, B, cfg.outer_tol, cfg.outer_max_iter, cfg.residual_history_stride, precond, lv.v,
               lv.cs, lv.ws, rep, s);
}

std::vector<double> lame_per_element(const Mesh& m, int32_t n_mat, const double* x) {
  std::vector<double> out(m.n_elems());
  for (int32_t e = 0; e < m.n_elems(); ++e) {
    const int32_t mid = m.material_id[e];
    if (mid < 0 || mid >= n_mat)
      validation("ebe: element " + std::to_string(e) + " references material " + std::to_string(mid) +
                 " but only " + std::to_string(n_mat) + " defined");
    out[e] = x[mid];
  }
  return out;
}

ts_levels* levels_create(const Mesh& m, int32_t n_mat, const double* lam, const double* mu, const uint8_t* dof_mask,
                         const ts_solver_config& cfg) {
  const auto t0 = clk::now();
  check_cfg(&cfg);
  require_device();
  auto lv = std::make_unique<ts_levels>();
  const int32_t N = m.n_nodes(), V = m.vertex_count;
  std::vector<uint8_t> mask0 = dof_mask ? std::vector<uint8_t>(dof_mask, dof_mask + 3 * size_t(N)) : m.dirichlet_mask();
  std::vector<uint8_t> mask1(mask0.begin(), mask0.begin() + 3 * size_t(V));
  lv->n0 = N;
  lv->n1 = V;
  setup_mark("levels: start");
  {
    const char* e = std::getenv("TSGPU_L1");
    lv->l1_assembled = !(e && std::string(e) == "ebe");
  }
  std::vector<int32_t> eorder;  // one Morton element order for the three operators
  PairTopology pairs;              // and one face-pair matching for the two tet10 operators
  lv->outer.reset(ebe_create(m, 2, n_mat, lam, mu, mask0.data(), 64, nullptr, -1, &eorder, &pairs));
  setup_mark("levels: outer operator");
  lv->l0.reset(ebe_create(m, 2, n_mat, lam, mu, mask0.data(), 32, nullptr, -1, &eorder, &pairs));
  // with the assembled level 1 the tet4 EBE operator only serves the API and its
  // block-Jacobi diagonal: no sweep plans
  lv->l1.reset(ebe_create(m, 1, n_mat, lam, mu, mask1.data(), 32, nullptr, lv->l1_assembled ? 3 : -1, &eorder));
  setup_mark("levels: l0 + l1 operators");
  // geometric P1 (prolongation.hpp:67-98): edge endpoints (vmin, vmax) + transpose
  {
    static constexpr int ee[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
    std::vector<int32_t> ends(2 * size_t(N - V), -1);
    // parallel fill (an edge shared by several elements is written with the same endpoints by each);
    // the first bad element, if any, is then reported as the sequential scan would
    int32_t first_bad = INT32_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
    for (int32_t e = 0; e < m.n_elems(); ++e) {
      const int32_t* t = m.tets10.data() + 10 * size_t(e);
      for (int q = 0; q < 6; ++q) {
        int32_t a = t[ee[q][0]], b = t[ee[q][1]];
        if (a > b) std::swap(a, b);
        const int32_t mid = t[4 + q];
        if (mid < V || a >= V || b >= V) {
          first_bad = std::min(first_bad, e);
          break;
        }
        __atomic_store_n(&ends[2 * size_t(mid - V)], a, __ATOMIC_RELAXED);
        __atomic_store_n(&ends[2 * size_t(mid - V) + 1], b, __ATOMIC_RELAXED);
      }
    }
    if (first_bad != INT32_MAX) {
      const int32_t* t = m.tets10.data() + 10 * size_t(first_bad);
      for (int q = 0; q < 6; ++q) {
        const int32_t a = t[ee[q][0]], b = t[ee[q][1]], mid = t[4 + q];
        if (mid < V) validation("geometric prolongation: edge node " + std::to_string(mid) + " is a vertex id");
        if (a >= V || b >= V) validation("geometric prolongation: edge endpoints must be vertices");
      }
    }
    std::vector<int32_t> tptr(V + 1, 0);
    for (int32_t k = 0; k < N - V; ++k) {
      if (ends[2 * size_t(k)] < 0)
        validation("geometric prolongation: edge node " + std::to_string(k + V) + " not present in edge map");
      ++tptr[ends[2 * size_t(k)] + 1];
      ++tptr[ends[2 * size_t(k) + 1] + 1];
    }
    for (int32_t i = 0; i < V; ++i) tptr[i + 1] += tptr[i];
    std::vector<int32_t> tidx(tptr[V]), cur(tptr.begin(), tptr.end() - 1);
    for (int32_t k = 0; k < N - V; ++k) {  // ascending fine node id
      tidx[cur[ends[2 * size_t(k)]]++] = k + V;
      tidx[cur[ends[2 * size_t(k) + 1]]++] = k + V;
    }
    lv->p1_ends.upload(ends);
    lv->p1t_ptr.upload(tptr);
    lv->p1t_idx.upload(tidx);
  }
  // K1 -> aggregation -> Galerkin level 2 (adaptive_cg.hpp:53-60)
  const std::vector<double> lam_e = lame_per_element(m, n_mat, lam), mu_e = lame_per_element(m, n_mat, mu);
  setup_mark("levels: P1");
  HostVec<float> k1f;  // the fp32 level-1 operator, float-rounded inputs, same pattern
  const BcsrD k1 = assemble_tet4(m, lam_e, mu_e, mask1, lv->l1_assembled ? &k1f : nullptr);
  setup_mark("levels: K1 assembly");
  if (lv->l1_assembled) {
    lv->l1_row_ptr.upload(k1.row_ptr);
    lv->l1_col_idx.upload(k1.col_idx);
    lv->l1_blocks.upload(k1f);
    setup_mark("levels: K1 fp32 operator");
  }
  Aggregation agg = aggregate_p1(k1, cfg.aggregate_target);
  setup_mark("levels: aggregation");
  const BcsrD a2 = build_level2(k1, agg, mask1);
  setup_mark("levels: Galerkin level 2");
  lv->n2 = agg.n_aggregates;
  lv->h_mask2 = coarse_mask(agg, mask1);
  lv->h_m2 = bcsr_block_jacobi_f32(a2);
  lv->h_agg = agg.agg_of_node;
  lv->h_seeds = agg.seeds;
  lv->h_rp2 = a2.row_ptr;
  lv->h_ci2.assign(a2.col_idx.begin(), a2.col_idx.end());
  lv->h_bl2.resize(a2.blocks.size());
  for (size_t q = 0; q < a2.blocks.size(); ++q) lv->h_bl2[q] = static_cast<float>(a2.blocks[q]);
  {
    std::vector<int32_t> aptr(lv->n2 + 1, 0), amem(V);
    for (int32_t r = 0; r < V; ++r) ++aptr[agg.agg_of_node[r] + 1];
    for (int32_t i = 0; i < lv->n2; ++i) aptr[i + 1] += aptr[i];
    std::vector<int32_t> cur(aptr.begin(), aptr.end() - 1);
    for (int32_t r = 0; r < V; ++r) amem[cur[agg.agg_of_node[r]]++] = r;
    lv->p2t_ptr.upload(aptr);
    lv->p2t_idx.upload(amem);
  }
  lv->agg.upload(lv->h_agg);
  lv->l2_row_ptr.upload(lv->h_rp2);
  lv->l2_col_idx.upload(lv->h_ci2);
  lv->l2_blocks.upload(lv->h_bl2);
  lv->m2.upload(lv->h_m2);
  lv->mask0.upload(mask0);
  lv->mask1.upload(mask1);
  lv->mask2.upload(lv->h_mask2);
  lv->m0.alloc(9 * size_t(N));
  lv->m1.alloc(9 * size_t(V));
  setup_mark("levels: uploads");
  ebe_block_jacobi(*lv->l0, lv->m0.get(), nullptr);
  ebe_block_jacobi(*lv->l1, lv->m1.get(), nullptr);
  // host setup copies no longer needed by the operators
  for (ts_ebe* op : {lv->l0.get(), lv->l1.get()}) {  // outer keeps them for solve_pcge's block Jacobi
    HostVec<double>().swap(op->coef64);
  }
  TS_CUDA(cudaDeviceSynchronize());
  setup_mark("levels: block Jacobi");
  lv->setup_s = secs(t0, clk::now());
  return lv.release();
}

}  // namespace

// entry points for other translation units (greens.cu)
ts_levels* levels_build(const Mesh& m, int32_t n_mat, const double* lam, const double* mu, const uint8_t* dof_mask,
                        const ts_solver_config& cfg) {
  return levels_create(m, n_mat, lam, mu, dof_mask, cfg);
}
void levels_free(ts_levels* lv) { delete lv; }
void levels_solve_device(ts_levels& lv, const double* f, const double* u0, double* u, int32_t B,
                         const ts_solver_config& cfg, ts_solve_report& rep, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(lv.mu);
  solve_device(lv, f, u0, u, B, cfg, rep, s);
}
int32_t levels_nodes(const ts_levels& lv) { return lv.n0; }
const uint8_t* levels_mask0(const ts_levels& lv) { return lv.mask0.get(); }
}  // namespace tsg

#define TS_API_BEGIN try {
#define TS_API_END                                   \
  }                                                  \
  catch (const tsg::Error& e) {                      \
    tsg::set_last_error(e.what());                   \
    return e.code;                                   \
  }                                                  \
  catch (const std::exception& e) {                  \
    tsg::set_last_error(e.what());                   \
    return TS_ERR_VALIDATION;                        \
  }                                                  \
  return TS_OK;

extern "C" {

ts_status ts_levels_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda, const double* mu,
                           const uint8_t* dof_mask, const ts_solver_config* cfg, ts_levels** out) {
  TS_API_BEGIN
  if (!mesh || !lambda || !mu || !cfg || !out) tsg::validation("levels: null argument");
  *out = tsg::levels_create(mesh->m, n_materials, lambda, mu, dof_mask, *cfg);
  TS_API_END
}

void ts_levels_destroy(ts_levels* lv) { delete lv; }

ts_status ts_levels_sizes(const ts_levels* lv, int32_t* n0, int32_t* n1, int32_t* n2, int64_t* nnzb2) {
  TS_API_BEGIN
  if (!lv) tsg::validation("levels: null handle");
  if (n0) *n0 = lv->n0;
  if (n1) *n1 = lv->n1;
  if (n2) *n2 = lv->n2;
  if (nnzb2) *nnzb2 = static_cast<int64_t>(lv->h_ci2.size());
  TS_API_END
}

ts_status ts_levels_export(const ts_levels* lv, int32_t* agg, int32_t* row_ptr2, int32_t* col_idx2, float* blocks2,
                           uint8_t* mask2, float* m2_inv) {
  TS_API_BEGIN
  if (!lv) tsg::validation("levels: null handle");
  if (agg) std::memcpy(agg, lv->h_agg.data(), lv->h_agg.size() * sizeof(int32_t));
  if (row_ptr2) std::memcpy(row_ptr2, lv->h_rp2.data(), lv->h_rp2.size() * sizeof(int32_t));
  if (col_idx2) std::memcpy(col_idx2, lv->h_ci2.data(), lv->h_ci2.size() * sizeof(int32_t));
  if (blocks2) std::memcpy(blocks2, lv->h_bl2.data(), lv->h_bl2.size() * sizeof(float));
  if (mask2) std::memcpy(mask2, lv->h_mask2.data(), lv->h_mask2.size());
  if (m2_inv) std::memcpy(m2_inv, lv->h_m2.data(), lv->h_m2.size() * sizeof(float));
  TS_API_END
}

ts_status ts_levels_export_fine(const ts_levels* lv, float* m0_inv, float* m1_inv, uint8_t* mask0, uint8_t* mask1,
                                int32_t* seeds) {
  TS_API_BEGIN
  if (!lv) tsg::validation("levels: null handle");
  if (m0_inv) TS_CUDA(cudaMemcpy(m0_inv, lv->m0.get(), 9 * size_t(lv->n0) * sizeof(float), cudaMemcpyDeviceToHost));
  if (m1_inv) TS_CUDA(cudaMemcpy(m1_inv, lv->m1.get(), 9 * size_t(lv->n1) * sizeof(float), cudaMemcpyDeviceToHost));
  if (mask0) TS_CUDA(cudaMemcpy(mask0, lv->mask0.get(), 3 * size_t(lv->n0), cudaMemcpyDeviceToHost));
  if (mask1) TS_CUDA(cudaMemcpy(mask1, lv->mask1.get(), 3 * size_t(lv->n1), cudaMemcpyDeviceToHost));
  if (seeds) std::memcpy(seeds, lv->h_seeds.data(), lv->h_seeds.size() * sizeof(int32_t));
  TS_API_END
}

ts_status ts_levels_operator(const ts_levels* lv, int32_t which, const ts_ebe** op) {
  TS_API_BEGIN
  if (!lv || !op) tsg::validation("levels: null argument");
  if (which == 0) *op = lv->outer.get();
  else if (which == 1) *op = lv->l0.get();
  else if (which == 2) *op = lv->l1.get();
  else tsg::validation("levels: operator index must be 0 (outer), 1 (level0) or 2 (level1)");
  TS_API_END
}

ts_status ts_levels_apply(ts_levels* lv, int32_t which, const void* u, void* f, int32_t batch, void* stream) {
  TS_API_BEGIN
  if (!lv || !u || !f) tsg::validation("levels apply: null argument");
  if (batch < 1) tsg::validation("levels apply: batch must be >= 1");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (which == 0) tsg::ebe_apply(*lv->outer, u, f, batch, s);
  else if (which == 1) tsg::ebe_apply(*lv->l0, u, f, batch, s);
  else if (which == 2 && lv->l1_assembled)
    tsg::bcsr_rows_f32(lv->l1_row_ptr.get(), lv->l1_col_idx.get(), lv->l1_blocks.get(), lv->n1,
                       static_cast<const float*>(u), static_cast<float*>(f), batch, s, nullptr,
                       static_cast<int64_t>(lv->l1_col_idx.size()));
  else if (which == 2) tsg::ebe_apply(*lv->l1, u, f, batch, s);
  else if (which == 3)
    tsg::bcsr_apply_f32(lv->l2_row_ptr.get(), lv->l2_col_idx.get(), lv->l2_blocks.get(), lv->n2,
                        static_cast<const float*>(u), static_cast<float*>(f), batch, s,
                        static_cast<int64_t>(lv->l2_col_idx.size()));
  else tsg::validation("levels apply: operator index must be 0 (outer), 1 (level0), 2 (level1) or 3 (level2)");
  TS_API_END
}

ts_status ts_levels_transfer(ts_levels* lv, int32_t which, const float* in, float* out, int32_t batch, void* stream) {
  TS_API_BEGIN
  if (!lv || !in || !out) tsg::validation("levels transfer: null argument");
  if (batch < 1) tsg::validation("levels transfer: batch must be >= 1");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (which) {
    case 0: tsg::p1_apply(in, out, lv->p1_ends.get(), lv->n1, lv->n0, lv->mask0.get(), batch, s); break;
    case 1:
      tsg::p1_restrict(in, out, lv->p1t_ptr.get(), lv->p1t_idx.get(), lv->n1, lv->mask1.get(), batch, s);
      break;
    case 2: tsg::p2_apply(in, out, lv->agg.get(), lv->n1, lv->mask1.get(), batch, s); break;
    case 3:
      tsg::p2_restrict(in, out, lv->p2t_ptr.get(), lv->p2t_idx.get(), lv->n2, lv->mask2.get(), batch, s);
      break;
    default: tsg::validation("levels transfer: which must be 0 (P1), 1 (P1^T), 2 (P2) or 3 (P2^T)");
  }
  TS_API_END
}

ts_status ts_solve_device(ts_levels* lv, const double* f, const double* u0, double* u_out, int32_t n_nodes,
                          int32_t batch, const ts_solver_config* cfg, ts_solve_report* rep, void* stream) {
  TS_API_BEGIN
  if (!lv || !f || !u0 || !u_out || !cfg) tsg::validation("solve: null argument");
  if (n_nodes != lv->n0) tsg::validation("solve: dimension mismatch");
  ts_solve_report local{};
  ts_solve_report& r = rep ? *rep : local;
  std::lock_guard<std::mutex> lock(lv->mu);
  tsg::solve_device(*lv, f, u0, u_out, batch, *cfg, r, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_solve(ts_levels* lv, const double* f, const double* u0, double* u_out, int32_t n_nodes, int32_t batch,
                   const ts_solver_config* cfg, ts_solve_report* rep) {
  TS_API_BEGIN
  if (!lv || !f || !u0 || !u_out || !cfg) tsg::validation("solve: null argument");
  if (n_nodes != lv->n0) tsg::validation("solve: dimension mismatch");
  if (batch < 1) tsg::validation("solve: batch must be >= 1");
  ts_solve_report local{};
  ts_solve_report& r = rep ? *rep : local;
  std::lock_guard<std::mutex> lock(lv->mu);
  const size_t bytes = 3 * size_t(lv->n0) * batch * sizeof(double);
  DevBuf<double>& df = lv->host_f;
  DevBuf<double>& du = lv->host_u;
  df.ensure(bytes / 8);
  du.ensure(bytes / 8);
  cudaStream_t s = nullptr;
  TS_CUDA(cudaMemcpyAsync(df.get(), f, bytes, cudaMemcpyHostToDevice, s));
  TS_CUDA(cudaMemcpyAsync(du.get(), u0, bytes, cudaMemcpyHostToDevice, s));
  ts_status rc = TS_OK;
  std::string msg;
  try {
    tsg::solve_device(*lv, df.get(), du.get(), du.get(), batch, *cfg, r, s);
  } catch (const tsg::Error& e) {
    rc = e.code;
    msg = e.what();
  }
  if (rc == TS_OK || rc == TS_ERR_NO_CONVERGENCE)
    TS_CUDA(cudaMemcpy(u_out, du.get(), bytes, cudaMemcpyDeviceToHost));
  if (rc != TS_OK) tsg::fail(rc, msg);
  TS_API_END
}

ts_status ts_solve_pcge(const ts_ebe* k, const double* f, const double* u0, double* u_out, int32_t n_nodes,
                        int32_t batch, double tol, int32_t max_iter, ts_solve_report* rep) {
  TS_API_BEGIN
  if (!k || !f || !u0 || !u_out) tsg::validation("solve_pcge: null argument");
  if (n_nodes != k->n_nodes) tsg::validation("ebe apply: dimension mismatch");
  if (k->prec != 64 || k->order != 2) tsg::validation("solve_pcge: needs the 64-bit second-order operator");
  if (batch < 1 || batch > tsg::kRedThreads) tsg::validation("solve_pcge: batch must be in [1, 256]");
  ts_solve_report local{};
  ts_solve_report& r = rep ? *rep : local;
  tsg::report_reset(r, 1, 64);
  const int32_t n = k->n_nodes;
  const size_t len = 3 * size_t(n) * batch;
  LevelVecs v;
  for (auto* b : {&v.r, &v.q, &v.z, &v.p, &v.scratch, &v.f, &v.u}) b->alloc(len);
  ColScalars cs;
  cs.ensure(batch);
  tsg::Workspace ws;
  ws.ensure(batch);
  DevBuf<double> m64(9 * size_t(n));
  cudaStream_t s = nullptr;
  tsg::ebe_block_jacobi(*k, m64.get(), s);
  TS_CUDA(cudaMemcpyAsync(v.f.get(), f, len * sizeof(double), cudaMemcpyHostToDevice, s));
  TS_CUDA(cudaMemcpyAsync(v.u.get(), u0, len * sizeof(double), cudaMemcpyHostToDevice, s));
  auto precond = [&](const double* rr, double* z) { tsg::bj_apply<double>(m64.get(), rr, z, n, batch, s); };
  ts_status rc = TS_OK;
  std::string msg;
  try {
    auto kop = [&](const double* x, double* y) { tsg::ebe_apply(*k, x, y, batch, s); };
    tsg::core::run_outer_cg(kop, k->n_nodes, v.f.get(), v.u.get(), batch, tol, max_iter, 0, precond, v, cs, ws, r, s);
  } catch (const tsg::Error& e) {
    rc = e.code;
    msg = e.what();
  }
  if (rc == TS_OK || rc == TS_ERR_NO_CONVERGENCE)
    TS_CUDA(cudaMemcpy(u_out, v.u.get(), len * sizeof(double), cudaMemcpyDeviceToHost));
  if (rc != TS_OK) tsg::fail(rc, msg);
  TS_API_END
}

}  // extern "C"
