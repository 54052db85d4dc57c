// greens.cu — the Green's-function bank on the device:
// compute_greens_bank (greens.hpp:114-145) = for each batch of B unit slips
// (greens_batch_plan, greens.hpp:102-110): lift the slips to right-hand sides
// (slip_to_rhs, fault.hpp:363-388: ONE multi-case fp64 EBE product on the
// split mesh for the whole batch), solve the batch (adaptive_cg.hpp:242-263),
// sample every observation (greens.hpp:50-76: first containing element, tet10
// shape values — located once, then a device gather for all columns).
#include <climits>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ebe.h"
#include "fault.h"
#include "dist_api.h"
#include "levels_api.h"

#include <algorithm>

namespace tsg {
namespace {

// g[plus][a][j] = +delta/2, g[minus][a][j] = -delta/2 (fault.hpp:370-376); d: [ns][3][W]
__global__ void k_slip_jump(const int32_t* __restrict__ plus, const int32_t* __restrict__ minus, int32_t ns, int32_t W,
                            const double* __restrict__ d, double* __restrict__ g) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(ns) * 3 * W) return;
  const int64_t k = i / (3 * W), rem = i - k * 3 * W;
  g[3 * int64_t(plus[k]) * W + rem] = 0.5 * d[i];
  g[3 * int64_t(minus[k]) * W + rem] = -0.5 * d[i];
}

// f[base] = -(w[first copy]) - w[second copy]; constrained base dofs zeroed (fault.hpp:380-386)
__global__ void k_lift(const double* __restrict__ w, const int32_t* __restrict__ s1, const int32_t* __restrict__ s2,
                       const uint8_t* __restrict__ mask, int32_t n, int32_t W, double* __restrict__ f) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(n) * 3 * W) return;
  const int64_t node = i / (3 * W), rem = i - node * 3 * W;
  double v = 0.0 - w[3 * int64_t(s1[node]) * W + rem];
  if (s2[node] >= 0) v -= w[3 * int64_t(s2[node]) * W + rem];
  f[i] = (mask && mask[3 * node + rem / W]) ? 0.0 : v;
}

// partitioned lift: local row i of f from the band products of its base node's split
// copies (l1 / l2 band indices, -1 = not in the band: no contribution), as k_lift
__global__ void k_lift_local(const double* __restrict__ w, const int32_t* __restrict__ l1,
                             const int32_t* __restrict__ l2, const uint8_t* __restrict__ mask, int32_t n, int32_t W,
                             double* __restrict__ f) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(n) * 3 * W) return;
  const int64_t node = i / (3 * W), rem = i - node * 3 * W;
  const int32_t a = l1[node], b = l2[node];
  double v = 0.0 - (a >= 0 ? w[3 * int64_t(a) * W + rem] : 0.0);
  if (b >= 0) v -= w[3 * int64_t(b) * W + rem];
  f[i] = (mask && mask[3 * node + rem / W]) ? 0.0 : v;
}

// bank[r][col0 + j] = sum_a n_a u[3 node_a + axis][j] (greens.hpp:70-73)
__global__ void k_sample(const double* __restrict__ u, const int32_t* __restrict__ nodes, const double* __restrict__ sh,
                         const int32_t* __restrict__ axis, int32_t n_obs, int32_t W, int32_t n_cols, int32_t col0,
                         double* __restrict__ bank) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(n_obs) * W) return;
  const int32_t r = static_cast<int32_t>(i / W), j = static_cast<int32_t>(i - int64_t(r) * W);
  double v = 0.0;
  if (axis[r] < 0) {  // partitioned sweep: the observation's element lives on another rank
    bank[int64_t(r) * n_cols + col0 + j] = 0.0;
    return;
  }
  for (int a = 0; a < 10; ++a) v += sh[10 * r + a] * u[(3 * int64_t(nodes[10 * r + a]) + axis[r]) * W + j];
  bank[int64_t(r) * n_cols + col0 + j] = v;
}

// reconstruct_split_solution (fault.hpp:392-411): u_split[s] = u_base[to_base[s]] ...
__global__ void k_split_gather(const double* __restrict__ ub, const int32_t* __restrict__ to_base, int32_t ns_nodes,
                               int32_t W, double* __restrict__ us) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(ns_nodes) * 3 * W) return;
  const int64_t s = i / (3 * W), rem = i - s * 3 * W;
  us[i] = ub[3 * int64_t(__ldg(to_base + s)) * W + rem];
}
// ... then plus copies += delta/2, minus copies -= delta/2 (in that order, as the reference)
__global__ void k_split_jump(const int32_t* __restrict__ plus, const int32_t* __restrict__ minus, int32_t ns, int32_t W,
                             const double* __restrict__ d, double* __restrict__ us) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(ns) * 3 * W) return;
  const int64_t k = i / (3 * W), rem = i - k * 3 * W;
  const double h = 0.5 * d[i];
  us[3 * int64_t(plus[k]) * W + rem] += h;
  us[3 * int64_t(minus[k]) * W + rem] -= h;
}

// IEEE ops without contraction: the device scan reproduces the host arithmetic
// of the reference's point location (greens.hpp:50-76, geometry.hpp:27-42) operation for operation
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// sample_displacement's point location (greens.hpp:50-76): the FIRST element (lowest id)
// containing each point, barycentric tolerance -1e-8. One thread per element tests every
// point; best[p] = atomicMin over containing elements. tet4 = the vertex ids of each element.
__global__ void k_locate(const double* __restrict__ xyz, const int32_t* __restrict__ tet4, int32_t E,
                         const double* __restrict__ pts, int32_t n, int32_t* __restrict__ best) {
  const int32_t e = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (e >= E) return;
  double v[4][3];
  for (int a = 0; a < 4; ++a) {
    const int64_t id = __ldg(tet4 + 4 * int64_t(e) + a);
    for (int c = 0; c < 3; ++c) v[a][c] = __ldg(xyz + 3 * id + c);
  }
  double m[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) m[r][c] = ds(v[c + 1][r], v[0][r]);
  // invert3 (geometry.hpp:27-42), same operation order as the host
  const double d = da(ds(dm(m[0][0], ds(dm(m[1][1], m[2][2]), dm(m[1][2], m[2][1]))),
                         dm(m[0][1], ds(dm(m[1][0], m[2][2]), dm(m[1][2], m[2][0])))),
                      dm(m[0][2], ds(dm(m[1][0], m[2][1]), dm(m[1][1], m[2][0]))));
  if (d == 0.0) return;
  const double id = __ddiv_rn(1.0, d);
  double inv[3][3];
  inv[0][0] = dm(ds(dm(m[1][1], m[2][2]), dm(m[1][2], m[2][1])), id);
  inv[0][1] = dm(ds(dm(m[0][2], m[2][1]), dm(m[0][1], m[2][2])), id);
  inv[0][2] = dm(ds(dm(m[0][1], m[1][2]), dm(m[0][2], m[1][1])), id);
  inv[1][0] = dm(ds(dm(m[1][2], m[2][0]), dm(m[1][0], m[2][2])), id);
  inv[1][1] = dm(ds(dm(m[0][0], m[2][2]), dm(m[0][2], m[2][0])), id);
  inv[1][2] = dm(ds(dm(m[0][2], m[1][0]), dm(m[0][0], m[1][2])), id);
  inv[2][0] = dm(ds(dm(m[1][0], m[2][1]), dm(m[1][1], m[2][0])), id);
  inv[2][1] = dm(ds(dm(m[0][1], m[2][0]), dm(m[0][0], m[2][1])), id);
  inv[2][2] = dm(ds(dm(m[0][0], m[1][1]), dm(m[0][1], m[1][0])), id);
  constexpr double kTol = -1e-8;
  for (int32_t q = 0; q < n; ++q) {
    const double d0 = ds(__ldg(pts + 3 * q), v[0][0]), d1 = ds(__ldg(pts + 3 * q + 1), v[0][1]),
                 d2 = ds(__ldg(pts + 3 * q + 2), v[0][2]);
    double xi[3];
    for (int r = 0; r < 3; ++r) xi[r] = da(da(dm(inv[r][0], d0), dm(inv[r][1], d1)), dm(inv[r][2], d2));
    const double l0 = ds(ds(ds(1.0, xi[0]), xi[1]), xi[2]);
    if (xi[0] < kTol || xi[1] < kTol || xi[2] < kTol || l0 < kTol) continue;
    atomicMin(best + q, e);
  }
}

}  // namespace
}  // namespace tsg

// FaultedModel (model.hpp:34-56) on the device
struct ts_faulted {
  tsg::Mesh base;        // host copy for point location
  tsg::Mesh split;
  tsg::FaultPatch patch;
  ts_levels* levels = nullptr;
  std::unique_ptr<ts_ebe> split_raw;  // unmasked fp64 tet10 on the split mesh
  tsg::DevBuf<int32_t> plus, minus, s1, s2;
  tsg::DevBuf<double> loc_xyz;    // base vertex coordinates (device point location)
  tsg::DevBuf<int32_t> loc_tet4;  // base element vertex ids
  tsg::DevBuf<double> bf, bu0, bu;  // per-batch f, u0, u of the bank loop (kept across calls)
  tsg::DevBuf<double> sg, sw;       // split-mesh work vectors of slip_to_rhs (kept across calls)
  tsg::DevBuf<int32_t> to_base;     // split node -> base node (reconstruct_split_solution)
  ~ts_faulted() { tsg::levels_free(levels); }
};

// The Green's-function bank on a PARTITIONED base mesh (configs[4] over the GPUs of
// one box): every rank holds the fault patch (split_nodes of the global mesh is
// cheap host work, computed identically everywhere), its partition's level set
// (ts_dist_levels), and the FAULT BAND of the split mesh — the elements that touch
// a split node, the only ones whose products with a slip jump are non-zero — so
// slip lifting is one small fp64 EBE product replicated on every rank, lifted onto
// the rank's own rows without communication. Each observation is sampled by the
// rank owning its (first containing) element; one all-reduce at the end assembles
// the bank on every rank.
struct ts_dist_faulted {
  tsg::Mesh base;            // global base mesh (point location, shape values)
  tsg::FaultPatch patch;
  ts_dist_levels* levels = nullptr;
  tsg::Comm* comm = nullptr;
  std::vector<int32_t> part;     // element -> rank
  std::vector<int32_t> l2g;      // local -> global node (ascending)
  std::unique_ptr<ts_ebe> band;  // unmasked fp64 tet10 on the fault band of the split mesh
  int32_t n_band = 0;
  tsg::DevBuf<int32_t> bplus, bminus;  // split copies, band numbering
  tsg::DevBuf<int32_t> lift1, lift2;   // local node -> band index of its base node's split copies (-1 none)
  tsg::DevBuf<double> loc_xyz;
  tsg::DevBuf<int32_t> loc_tet4;
  tsg::DevBuf<double> bg, bw, bf, bu0, bu;
  ~ts_dist_faulted() { tsg::dist_levels_destroy(levels); }
};

namespace tsg {

ts_faulted* faulted_create(const Mesh& m, int32_t n_mat, const double* lam, const double* mu,
                           const std::vector<std::array<int32_t, 3>>& tris, const ts_solver_config& cfg) {
  auto F = std::make_unique<ts_faulted>();
  F->base = m;
  split_nodes(m, tris, F->split, F->patch);
  F->split_raw.reset(ebe_create(F->split, 2, n_mat, lam, mu, nullptr, 64));
  F->levels = levels_build(m, n_mat, lam, mu, nullptr, cfg);
  const size_t ns = F->patch.split_nodes.size();
  std::vector<int32_t> pl(ns), mi(ns), s1(m.n_nodes()), s2(m.n_nodes(), -1);
  for (size_t k = 0; k < ns; ++k) {
    pl[k] = F->patch.split_nodes[k].plus;
    mi[k] = F->patch.split_nodes[k].minus;
  }
  // base node -> its split copies in ascending split id (the reference's accumulation order)
  std::vector<int32_t> seen(m.n_nodes(), 0);
  for (size_t s = 0; s < F->patch.to_base.size(); ++s) {
    const int32_t b = F->patch.to_base[s];
    if (seen[b]++ == 0) s1[b] = static_cast<int32_t>(s);
    else s2[b] = static_cast<int32_t>(s);
  }
  F->plus.upload(pl);
  F->minus.upload(mi);
  F->s1.upload(s1);
  F->s2.upload(s2);
  TS_CUDA(cudaDeviceSynchronize());
  return F.release();
}

// first containing element of each point (-1 = outside), device scan over the base mesh
// (vertex coordinates / element vertex ids cached in loc_xyz / loc_tet4)
std::vector<int32_t> locate_points(const Mesh& m, DevBuf<double>& loc_xyz, DevBuf<int32_t>& loc_tet4, int32_t n,
                                   const double* points) {
  const int32_t E = m.n_elems(), V = m.vertex_count;
  if (loc_tet4.size() != 4 * size_t(E)) {
    std::vector<double> xyz(m.coords.begin(), m.coords.begin() + 3 * size_t(V));
    std::vector<int32_t> t4(4 * size_t(E));
    for (int32_t e = 0; e < E; ++e)
      for (int a = 0; a < 4; ++a) t4[4 * size_t(e) + a] = m.tets10[10 * size_t(e) + a];
    loc_xyz.upload(xyz);
    loc_tet4.upload(t4);
  }
  DevBuf<double> dp;
  dp.upload(points, 3 * size_t(n));
  DevBuf<int32_t> best(n);
  std::vector<int32_t> h(n, INT32_MAX);
  TS_CUDA(cudaMemcpy(best.get(), h.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (E > 0) {
    k_locate<<<grid_for(E, 128), 128>>>(loc_xyz.get(), loc_tet4.get(), E, dp.get(), n, best.get());
    TS_CUDA(cudaGetLastError());
  }
  TS_CUDA(cudaMemcpy(h.data(), best.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int32_t& x : h)
    if (x == INT32_MAX) x = -1;
  return h;
}

// delta (device [ns][3][W]) of W unit slips (slip_vectors, fault.hpp:347-361)
void slip_deltas(const FaultPatch& patch, const Mesh& base, int32_t W, const double* centers, const int32_t* dirs,
                 const double* radii, DevBuf<double>& d) {
  const size_t ns = patch.split_nodes.size();
  std::vector<double> h(ns * 3 * W);
  for (int32_t j = 0; j < W; ++j) {
    const V3 c = {centers[3 * j], centers[3 * j + 1], centers[3 * j + 2]};
    if (dirs[j] != 0 && dirs[j] != 1) validation("unit slip: direction must be 0 (dip) or 1 (strike)");
    const std::vector<double> mag = unit_slip_magnitudes(patch, base, c, radii[j]);
    for (size_t k = 0; k < ns; ++k) {
      const V3& dir = dirs[j] == 0 ? patch.split_nodes[k].dip : patch.split_nodes[k].strike;
      for (int a = 0; a < 3; ++a) h[(3 * k + a) * W + j] = mag[k] * dir[a];
    }
  }
  d.upload(h);
}

// f (device [N][3][W]) = slip_to_rhs of W unit slips
void slips_to_rhs(ts_faulted& F, int32_t W, const double* centers, const int32_t* dirs, const double* radii, double* f,
                  cudaStream_t s) {
  const int32_t ns = static_cast<int32_t>(F.patch.split_nodes.size());
  const int32_t NS = F.split.n_nodes(), N = F.base.n_nodes();
  DevBuf<double> d;
  DevBuf<double>&g = F.sg, &w = F.sw;  // split-mesh slip jumps / products, kept across calls
  g.ensure(3 * size_t(NS) * W);
  w.ensure(3 * size_t(NS) * W);
  slip_deltas(F.patch, F.base, W, centers, dirs, radii, d);
  TS_CUDA(cudaMemsetAsync(g.get(), 0, 3 * size_t(NS) * W * sizeof(double), s));
  k_slip_jump<<<grid_for(int64_t(ns) * 3 * W, 256), 256, 0, s>>>(F.plus.get(), F.minus.get(), ns, W, d.get(), g.get());
  TS_CUDA_LAUNCH();
  ebe_apply(*F.split_raw, g.get(), w.get(), W, s);
  k_lift<<<grid_for(int64_t(N) * 3 * W, 256), 256, 0, s>>>(w.get(), F.s1.get(), F.s2.get(), levels_mask0(*F.levels), N,
                                                             W, f);
  TS_CUDA_LAUNCH();
  TS_CUDA(cudaStreamSynchronize(s));
}

ts_dist_faulted* dist_faulted_create(const Mesh& m, int32_t n_mat, const double* lam, const double* mu,
                                     const std::vector<std::array<int32_t, 3>>& tris, const int32_t* part,
                                     const ts_solver_config& cfg, Comm* comm) {
  auto F = std::make_unique<ts_dist_faulted>();
  F->base = m;
  F->comm = comm;
  F->part.assign(part, part + m.n_elems());
  Mesh split;
  split_nodes(m, tris, split, F->patch);
  const int32_t NS = split.n_nodes(), N = m.n_nodes(), E = split.n_elems();
  // fault band: split-mesh elements touching a split copy, compactly renumbered
  std::vector<uint8_t> on(NS, 0);
  for (const SplitNode& sn : F->patch.split_nodes) on[sn.plus] = on[sn.minus] = 1;
  std::vector<int32_t> bid(NS, -1);
  Mesh bm;
  for (int32_t e = 0; e < E; ++e) {
    const int32_t* t = split.tets10.data() + 10 * size_t(e);
    bool touch = false;
    for (int a = 0; a < 10 && !touch; ++a) touch = on[t[a]] != 0;
    if (!touch) continue;
    for (int a = 0; a < 10; ++a) {
      if (bid[t[a]] < 0) {
        bid[t[a]] = static_cast<int32_t>(bm.coords.size() / 3);
        for (int c = 0; c < 3; ++c) bm.coords.push_back(split.coords[3 * size_t(t[a]) + c]);
      }
      bm.tets10.push_back(bid[t[a]]);
    }
    bm.material_id.push_back(split.material_id[e]);
  }
  bm.vertex_count = bm.n_nodes();
  F->n_band = bm.n_nodes();
  F->band.reset(ebe_create(bm, 2, n_mat, lam, mu, nullptr, 64));
  const size_t ns = F->patch.split_nodes.size();
  std::vector<int32_t> pl(ns), mi(ns);
  for (size_t k = 0; k < ns; ++k) {
    pl[k] = bid[F->patch.split_nodes[k].plus];
    mi[k] = bid[F->patch.split_nodes[k].minus];
  }
  F->bplus.upload(pl);
  F->bminus.upload(mi);
  // base node -> its split copies in ascending split id (the reference's accumulation order), as band ids
  std::vector<int32_t> s1(N, -1), s2(N, -1);
  {
    std::vector<uint8_t> seen(N, 0);
    for (size_t q = 0; q < F->patch.to_base.size(); ++q) {
      const int32_t b = F->patch.to_base[q];
      (seen[b]++ == 0 ? s1[b] : s2[b]) = bid[q];
    }
  }
  split = Mesh();
  F->levels = dist_levels_create(m, n_mat, lam, mu, nullptr, part, cfg, comm);
  F->l2g = dist_local_nodes(*F->levels);
  const size_t nl = F->l2g.size();
  std::vector<int32_t> l1(nl), l2(nl);
  for (size_t i = 0; i < nl; ++i) {
    l1[i] = s1[F->l2g[i]];
    l2[i] = s2[F->l2g[i]];
  }
  F->lift1.upload(l1);
  F->lift2.upload(l2);
  TS_CUDA(cudaDeviceSynchronize());
  return F.release();
}

// this rank's rows (device [n_local][3][W]) of slip_to_rhs of W unit slips
void dist_slips_to_rhs(ts_dist_faulted& F, int32_t W, const double* centers, const int32_t* dirs, const double* radii,
                       double* f, cudaStream_t s) {
  const int32_t ns = static_cast<int32_t>(F.patch.split_nodes.size());
  const int32_t nl = static_cast<int32_t>(F.l2g.size());
  DevBuf<double> d;
  F.bg.ensure(3 * size_t(F.n_band) * W);
  F.bw.ensure(3 * size_t(F.n_band) * W);
  slip_deltas(F.patch, F.base, W, centers, dirs, radii, d);
  TS_CUDA(cudaMemsetAsync(F.bg.get(), 0, 3 * size_t(F.n_band) * W * sizeof(double), s));
  k_slip_jump<<<grid_for(int64_t(ns) * 3 * W, 256), 256, 0, s>>>(F.bplus.get(), F.bminus.get(), ns, W, d.get(),
                                                                  F.bg.get());
  TS_CUDA_LAUNCH();
  ebe_apply(*F.band, F.bg.get(), F.bw.get(), W, s);
  k_lift_local<<<grid_for(int64_t(nl) * 3 * W, 256), 256, 0, s>>>(F.bw.get(), F.lift1.get(), F.lift2.get(),
                                                                   dist_levels_mask0(*F.levels), nl, W, f);
  TS_CUDA_LAUNCH();
  TS_CUDA(cudaStreamSynchronize(s));
}

}  // namespace tsg

extern "C" {

ts_status ts_fault_plane_faces(const ts_mesh* mesh, int32_t axis, double coord, const double lo[3], const double hi[3],
                               int32_t* n_faces, int32_t* faces) {
  try {
    if (!mesh || !lo || !hi || !n_faces) tsg::validation("fault plane: null argument");
    const auto f = tsg::find_plane_fault_faces(mesh->m, axis, coord, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]});
    if (faces) {
      if (*n_faces < static_cast<int32_t>(f.size())) tsg::validation("fault plane: faces buffer too small");
      for (size_t i = 0; i < f.size(); ++i)
        for (int k = 0; k < 3; ++k) faces[3 * i + k] = f[i][k];
    }
    *n_faces = static_cast<int32_t>(f.size());
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

ts_status ts_faulted_model_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda, const double* mu,
                                  const int32_t* faces, int32_t n_faces, const ts_solver_config* cfg,
                                  ts_faulted** out) {
  try {
    if (!mesh || !lambda || !mu || !faces || !cfg || !out) tsg::validation("faulted model: null argument");
    if (n_faces < 1) tsg::validation("split_nodes: empty fault surface");
    if (ts_config_validate(cfg) != TS_OK) tsg::fail(TS_ERR_VALIDATION, ts_last_error());
    std::vector<std::array<int32_t, 3>> tris(n_faces);
    for (int32_t i = 0; i < n_faces; ++i)
      for (int k = 0; k < 3; ++k) tris[i][k] = faces[3 * i + k];
    *out = tsg::faulted_create(mesh->m, n_materials, lambda, mu, tris, *cfg);
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

void ts_faulted_model_destroy(ts_faulted* fm) { delete fm; }

ts_status ts_faulted_info(const ts_faulted* fm, int32_t* n_split_nodes, int32_t* split_mesh_nodes, int32_t* n_faces) {
  if (!fm) {
    tsg::set_last_error("faulted model: null handle");
    return TS_ERR_VALIDATION;
  }
  if (n_split_nodes) *n_split_nodes = static_cast<int32_t>(fm->patch.split_nodes.size());
  if (split_mesh_nodes) *split_mesh_nodes = fm->split.n_nodes();
  if (n_faces) *n_faces = static_cast<int32_t>(fm->patch.faces.size());
  return TS_OK;
}

ts_status ts_faulted_levels(const ts_faulted* fm, ts_levels** levels) {
  if (!fm || !levels) {
    tsg::set_last_error("faulted model: null argument");
    return TS_ERR_VALIDATION;
  }
  *levels = fm->levels;
  return TS_OK;
}

ts_status ts_reconstruct_split_solution(ts_faulted* fm, int32_t n_slips, const double* centers,
                                        const int32_t* directions, const double* radii, const double* u_base_host,
                                        double* u_split_host) {
  try {
    if (!fm || !centers || !directions || !radii || !u_base_host || !u_split_host)
      tsg::validation("reconstruct_split_solution: null argument");
    if (n_slips < 1) tsg::validation("reconstruct_split_solution: need at least one slip");
    const int32_t N = fm->base.n_nodes(), NS = fm->split.n_nodes();
    const int32_t ns = static_cast<int32_t>(fm->patch.split_nodes.size());
    if (fm->to_base.size() != size_t(NS)) fm->to_base.upload(fm->patch.to_base);
    tsg::DevBuf<double> ub, us(3 * size_t(NS) * n_slips), d;
    ub.upload(u_base_host, 3 * size_t(N) * n_slips);
    tsg::slip_deltas(fm->patch, fm->base, n_slips, centers, directions, radii, d);
    tsg::k_split_gather<<<tsg::grid_for(int64_t(NS) * 3 * n_slips, 256), 256>>>(ub.get(), fm->to_base.get(), NS,
                                                                               n_slips, us.get());
    TS_CUDA(cudaGetLastError());
    tsg::k_split_jump<<<tsg::grid_for(int64_t(ns) * 3 * n_slips, 256), 256>>>(fm->plus.get(), fm->minus.get(), ns,
                                                                            n_slips, d.get(), us.get());
    TS_CUDA(cudaGetLastError());
    TS_CUDA(cudaMemcpy(u_split_host, us.get(), us.size() * sizeof(double), cudaMemcpyDeviceToHost));
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

ts_status ts_slip_to_rhs(ts_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                         const double* radii, double* f_host) {
  try {
    if (!fm || !centers || !directions || !radii || !f_host) tsg::validation("slip_to_rhs: null argument");
    if (n_slips < 1) tsg::validation("slip_to_rhs: need at least one slip");
    const size_t len = 3 * size_t(fm->base.n_nodes()) * n_slips;
    tsg::DevBuf<double> f(len);
    tsg::slips_to_rhs(*fm, n_slips, centers, directions, radii, f.get(), nullptr);
    TS_CUDA(cudaMemcpy(f_host, f.get(), len * sizeof(double), cudaMemcpyDeviceToHost));
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

ts_status ts_greens_bank(ts_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                         const double* radii, int32_t n_obs, const double* points, const int32_t* axes,
                         const ts_solver_config* cfg, double* bank, int32_t* solver_calls, int64_t* outer_iterations) {
  try {
    if (!fm || !centers || !directions || !radii || !points || !axes || !cfg || !bank)
      tsg::validation("greens: null argument");
    if (n_slips < 1) tsg::validation("greens: need at least one unit slip");
    if (cfg->batch_size < 1) tsg::validation("greens: batch size must be >= 1");
    if (n_obs < 1) tsg::validation("greens: no observation components");
    const int32_t N = fm->base.n_nodes();
    // locate every observation once (the reference re-scans per column; same element, same
    // values): first containing element by a device scan, tet10 shape values on the host
    for (int32_t r = 0; r < n_obs; ++r)
      if (axes[r] < 0 || axes[r] > 2) tsg::validation("greens: observation axis must be 0..2");
    const std::vector<int32_t> elem = tsg::locate_points(fm->base, fm->loc_xyz, fm->loc_tet4, n_obs, points);
    std::vector<int32_t> nodes(10 * size_t(n_obs)), ax(n_obs);
    std::vector<double> sh(10 * size_t(n_obs));
    for (int32_t r = 0; r < n_obs; ++r) {
      const tsg::V3 p = {points[3 * r], points[3 * r + 1], points[3 * r + 2]};
      if (elem[r] < 0)
        tsg::validation("observation point (" + std::to_string(p[0]) + ", " + std::to_string(p[1]) + ", " +
                        std::to_string(p[2]) + ") lies outside the mesh");
      tsg::tet10_shape_at(fm->base, elem[r], p, sh.data() + 10 * r);
      for (int a = 0; a < 10; ++a) nodes[10 * r + a] = fm->base.tets10[10 * size_t(elem[r]) + a];
      ax[r] = axes[r];
    }
    tsg::DevBuf<int32_t> dn, da;
    tsg::DevBuf<double> ds, dbank(size_t(n_obs) * n_slips);
    dn.upload(nodes);
    da.upload(ax);
    ds.upload(sh);
    const int32_t B = cfg->batch_size;
    tsg::DevBuf<double>&f = fm->bf, &u0 = fm->bu0, &u = fm->bu;
    for (tsg::DevBuf<double>* b : {&f, &u0, &u}) b->ensure(3 * size_t(N) * B);
    int32_t calls = 0;
    int64_t outer = 0;
    for (int32_t lo = 0; lo < n_slips; lo += B) {  // greens_batch_plan (greens.hpp:102-110)
      const int32_t W = std::min(n_slips, lo + B) - lo;
      tsg::slips_to_rhs(*fm, W, centers + 3 * lo, directions + lo, radii + lo, f.get(), nullptr);
      TS_CUDA(cudaMemset(u0.get(), 0, 3 * size_t(N) * W * sizeof(double)));
      ts_solve_report rep{};
      tsg::levels_solve_device(*fm->levels, f.get(), u0.get(), u.get(), W, *cfg, rep, nullptr);
      ++calls;
      outer += rep.outer_iterations;
      tsg::k_sample<<<tsg::grid_for(int64_t(n_obs) * W, 256), 256>>>(u.get(), dn.get(), ds.get(), da.get(), n_obs, W,
                                                                      n_slips, lo, dbank.get());
      TS_CUDA(cudaGetLastError());
    }
    TS_CUDA(cudaMemcpy(bank, dbank.get(), dbank.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (solver_calls) *solver_calls = calls;
    if (outer_iterations) *outer_iterations = outer;
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

// ------------------------------------------------ partitioned Green's sweep (configs[4])

ts_status ts_dist_faulted_model_create(const ts_mesh* mesh, int32_t n_materials, const double* lambda,
                                       const double* mu, const int32_t* faces, int32_t n_faces, const int32_t* part,
                                       const ts_solver_config* cfg, ts_comm* comm, ts_dist_faulted** out) {
  tsg::Comm* c = comm ? tsg::comm_of(comm) : nullptr;
  try {
    if (!mesh || !lambda || !mu || !faces || !part || !cfg || !comm || !out)
      tsg::validation("dist faulted model: null argument");
    if (n_faces < 1) tsg::validation("split_nodes: empty fault surface");
    if (ts_config_validate(cfg) != TS_OK) tsg::fail(TS_ERR_VALIDATION, ts_last_error());
    std::vector<std::array<int32_t, 3>> tris(n_faces);
    for (int32_t i = 0; i < n_faces; ++i)
      for (int k = 0; k < 3; ++k) tris[i][k] = faces[3 * i + k];
    *out = tsg::dist_faulted_create(mesh->m, n_materials, lambda, mu, tris, part, *cfg, c);
  } catch (const tsg::Error& e) {
    if (c) c->abort();
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->abort();
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

void ts_dist_faulted_model_destroy(ts_dist_faulted* fm) { delete fm; }

ts_status ts_dist_faulted_levels(const ts_dist_faulted* fm, ts_dist_levels** levels) {
  if (!fm || !levels) {
    tsg::set_last_error("dist faulted model: null argument");
    return TS_ERR_VALIDATION;
  }
  *levels = fm->levels;
  return TS_OK;
}

ts_status ts_dist_slip_to_rhs(ts_dist_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                              const double* radii, double* f_local_host) {
  try {
    if (!fm || !centers || !directions || !radii || !f_local_host) tsg::validation("slip_to_rhs: null argument");
    if (n_slips < 1) tsg::validation("slip_to_rhs: need at least one slip");
    const size_t len = 3 * fm->l2g.size() * n_slips;
    tsg::DevBuf<double> f(len);
    tsg::dist_slips_to_rhs(*fm, n_slips, centers, directions, radii, f.get(), nullptr);
    TS_CUDA(cudaMemcpy(f_local_host, f.get(), len * sizeof(double), cudaMemcpyDeviceToHost));
  } catch (const tsg::Error& e) {
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

ts_status ts_dist_greens_bank(ts_dist_faulted* fm, int32_t n_slips, const double* centers, const int32_t* directions,
                              const double* radii, int32_t n_obs, const double* points, const int32_t* axes,
                              const ts_solver_config* cfg, double* bank, int32_t* solver_calls,
                              int64_t* outer_iterations) {
  tsg::Comm* c = fm ? fm->comm : nullptr;
  try {
    if (!fm || !centers || !directions || !radii || !points || !axes || !cfg || !bank)
      tsg::validation("greens: null argument");
    if (n_slips < 1) tsg::validation("greens: need at least one unit slip");
    if (cfg->batch_size < 1) tsg::validation("greens: batch size must be >= 1");
    if (n_obs < 1) tsg::validation("greens: no observation components");
    for (int32_t r = 0; r < n_obs; ++r)
      if (axes[r] < 0 || axes[r] > 2) tsg::validation("greens: observation axis must be 0..2");
    // the same first containing element on every rank (scan of the global mesh); its owner samples
    const std::vector<int32_t> elem = tsg::locate_points(fm->base, fm->loc_xyz, fm->loc_tet4, n_obs, points);
    const int rank = fm->comm->rank();
    std::vector<int32_t> nodes(10 * size_t(n_obs), 0), ax(n_obs, -1);
    std::vector<double> sh(10 * size_t(n_obs), 0.0);
    for (int32_t r = 0; r < n_obs; ++r) {
      const tsg::V3 p = {points[3 * r], points[3 * r + 1], points[3 * r + 2]};
      if (elem[r] < 0)
        tsg::validation("observation point (" + std::to_string(p[0]) + ", " + std::to_string(p[1]) + ", " +
                        std::to_string(p[2]) + ") lies outside the mesh");
      if (fm->part[elem[r]] != rank) continue;
      tsg::tet10_shape_at(fm->base, elem[r], p, sh.data() + 10 * r);
      for (int a = 0; a < 10; ++a) {
        const int32_t g = fm->base.tets10[10 * size_t(elem[r]) + a];
        const auto it = std::lower_bound(fm->l2g.begin(), fm->l2g.end(), g);
        if (it == fm->l2g.end() || *it != g) tsg::validation("greens: owned element node missing from partition");
        nodes[10 * r + a] = static_cast<int32_t>(it - fm->l2g.begin());
      }
      ax[r] = axes[r];
    }
    tsg::DevBuf<int32_t> dn, da;
    tsg::DevBuf<double> ds, dbank(size_t(n_obs) * n_slips);
    dn.upload(nodes);
    da.upload(ax);
    ds.upload(sh);
    const int32_t B = cfg->batch_size;
    const size_t nl = fm->l2g.size();
    for (tsg::DevBuf<double>* b : {&fm->bf, &fm->bu0, &fm->bu}) b->ensure(3 * nl * B);
    int32_t calls = 0;
    int64_t outer = 0;
    for (int32_t lo = 0; lo < n_slips; lo += B) {  // greens_batch_plan (greens.hpp:102-110)
      const int32_t W = std::min(n_slips, lo + B) - lo;
      tsg::dist_slips_to_rhs(*fm, W, centers + 3 * lo, directions + lo, radii + lo, fm->bf.get(), nullptr);
      TS_CUDA(cudaMemset(fm->bu0.get(), 0, 3 * nl * W * sizeof(double)));
      ts_solve_report rep{};
      tsg::dist_solve_device(*fm->levels, fm->bf.get(), fm->bu0.get(), fm->bu.get(), W, *cfg, rep, nullptr);
      ++calls;
      outer += rep.outer_iterations;
      tsg::k_sample<<<tsg::grid_for(int64_t(n_obs) * W, 256), 256>>>(fm->bu.get(), dn.get(), ds.get(), da.get(), n_obs,
                                                                      W, n_slips, lo, dbank.get());
      TS_CUDA(cudaGetLastError());
    }
    fm->comm->allreduce_sum(dbank.get(), dbank.size(), nullptr);  // each row from its owner, zeros elsewhere
    TS_CUDA(cudaMemcpy(bank, dbank.get(), dbank.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (solver_calls) *solver_calls = calls;
    if (outer_iterations) *outer_iterations = outer;
  } catch (const tsg::Error& e) {
    if (c && e.code != TS_ERR_NO_CONVERGENCE && e.code != TS_ERR_BREAKDOWN && e.code != TS_ERR_NONFINITE) c->abort();
    tsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->abort();
    tsg::set_last_error(e.what());
    return TS_ERR_VALIDATION;
  }
  return TS_OK;
}

}  // extern "C"
