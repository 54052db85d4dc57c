// dist_solver.cu — the partitioned multi-GPU solve: one rank
// per GPU (NCCL) or per host thread (in-process backend), each holding one
// element partition of the mesh.
//
//  * EBE products (K1/K2, ebe_operator.hpp:90-188): each rank sweeps its
//    partition's boundary elements first, then — while the interface rows'
//    partial sums travel to the neighbouring partitions (NCCL send/recv on a
//    side stream) — its interior elements; received partials are added in
//    ascending rank order so every copy of an interface node agrees bit for bit.
//  * Dot products (vector_batch.hpp:51-64) count each dof on its owner rank
//    and all-reduce the per-column fp64 sums (blas.cu finish_partials).
//  * Level 1 (tet4 on the vertex prefix) exchanges the same way; the
//    restrictions P1^T / P2^T sum owned fine rows only, then exchange
//    (level 1) or all-reduce (level 2). Level 2 — the Galerkin operator of the
//    reference's sequential aggregation (aggregation.hpp:23-185), built from
//    the global mesh exactly as on one device — is replicated: every rank runs
//    the identical level-2 PCG, so no communication happens inside it.
//  * Block-Jacobi diagonals of interface nodes are summed across ranks before
//    inversion (block_jacobi.hpp:45-66).
// The control loops are the single-device ones (solver_core.h), so the
// reference's recurrences, breakdown rules and termination tests apply
// unchanged to the global quantities.
#include <omp.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "dist.h"
#include "dist_api.h"
#include "setup.h"
#include "solver_core.h"

namespace tsg {
namespace {

using namespace core;

template <typename T>
__global__ void k_halo_pack(const T* __restrict__ x, const int32_t* __restrict__ rows, int64_t n, int W,
                            T* __restrict__ buf) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  const int64_t r = i / W;
  buf[i] = x[int64_t(rows[r]) * W + (i - r * W)];
}

// x[node] = sum over the node's sharing ranks, ascending rank order, of their
// partial rows (own partial in x, neighbours' in the receive buffer). Rows of
// constrained dofs keep their own value (every rank holds the identity row).
template <typename T>
__global__ void k_halo_sum(T* __restrict__ x, const int32_t* __restrict__ sh, int32_t nsh,
                           const int32_t* __restrict__ sptr, const int32_t* __restrict__ src,
                           const int64_t* __restrict__ roff, const T* __restrict__ rbuf, int W, int B,
                           const uint8_t* __restrict__ mask) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(nsh) * W) return;
  const int32_t k = static_cast<int32_t>(i / W);
  const int j = static_cast<int>(i - int64_t(k) * W);
  const int64_t node = sh[k];
  if (mask && mask[3 * node + j / B]) return;
  T acc = T(0);
  bool first = true;
  for (int32_t p = sptr[k]; p < sptr[k + 1]; ++p) {
    const int32_t sc = src[p];
    const T v = sc < 0 ? x[node * W + j] : rbuf[(roff[sc >> 24] + (sc & 0xFFFFFF)) * W + j];
    acc = first ? v : acc + v;
    first = false;
  }
  x[node * W + j] = acc;
}

// y[i] = x[rows[i]] over rows of width W (gather of this rank's coarse rows)
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ x, const int32_t* __restrict__ rows, int64_t n, int W,
                              T* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  const int64_t r = i / W;
  y[i] = x[int64_t(rows[r]) * W + (i - r * W)];
}
// x[rows[i]] = y[i] (scatter back into a zeroed full-length vector)
template <typename T>
__global__ void k_scatter_rows(const T* __restrict__ y, const int32_t* __restrict__ rows, int64_t n, int W,
                               T* __restrict__ x) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  const int64_t r = i / W;
  x[int64_t(rows[r]) * W + (i - r * W)] = y[i];
}

// Device image of a Halo plus its message buffers.
struct HaloDev {
  std::vector<int> nbr;
  std::vector<int64_t> roff;  // [nn + 1] first row of each neighbour
  DevBuf<int32_t> rows, sh, sptr, src;
  DevBuf<int64_t> roff_dev;
  int32_t nsh = 0;
  DevBuf<unsigned char> sbuf, rbuf;
  void build(const Halo& h) {
    nbr = h.nbr;
    roff.assign(1, 0);
    std::vector<int32_t> all;
    for (const auto& r : h.rows) {
      all.insert(all.end(), r.begin(), r.end());
      roff.push_back(static_cast<int64_t>(all.size()));
    }
    rows.upload(all);
    roff_dev.upload(roff);
    sh.upload(h.sh_nodes);
    sptr.upload(h.src_ptr);
    src.upload(h.src);
    nsh = static_cast<int32_t>(h.sh_nodes.size());
  }
  // rows of width W (T scalars) of x: exchange shared partials and sum them
  template <typename T>
  void run(T* x, int W, int B, const uint8_t* mask, Comm& comm, cudaStream_t s) {
    if (nbr.empty()) return;
    const int64_t nr = roff.back();
    const size_t bytes = size_t(nr) * W * sizeof(T);
    sbuf.ensure(bytes);
    rbuf.ensure(bytes);
    k_halo_pack<T><<<grid_for(nr * W, 256), 256, 0, s>>>(x, rows.get(), nr, W, reinterpret_cast<T*>(sbuf.get()));
    TS_CUDA_LAUNCH();
    const int nn = static_cast<int>(nbr.size());
    std::vector<void*> sp(nn), rp(nn);
    std::vector<size_t> sb(nn);
    for (int k = 0; k < nn; ++k) {
      sp[k] = sbuf.get() + size_t(roff[k]) * W * sizeof(T);
      rp[k] = rbuf.get() + size_t(roff[k]) * W * sizeof(T);
      sb[k] = size_t(roff[k + 1] - roff[k]) * W * sizeof(T);
    }
    comm.exchange(nn, nbr.data(), sp.data(), sb.data(), rp.data(), sb.data(), s);
    k_halo_sum<T><<<grid_for(int64_t(nsh) * W, 256), 256, 0, s>>>(x, sh.get(), nsh, sptr.get(), src.get(),
                                                                    roff_dev.get(), reinterpret_cast<const T*>(rbuf.get()),
                                                                    W, B, mask);
    TS_CUDA_LAUNCH();
  }
};

// A partition's EBE operator with its interface exchange.
struct DistEbe {
  std::unique_ptr<ts_ebe> op;
  HaloDev halo;
  const uint8_t* mask = nullptr;  // device, local dof mask of this level
  Comm* comm = nullptr;
  bool overlap = true;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_b = nullptr, ev_h = nullptr;
  ~DistEbe() {
    if (ev_b) cudaEventDestroy(ev_b);
    if (ev_h) cudaEventDestroy(ev_h);
    if (side) cudaStreamDestroy(side);
  }
  template <typename T>
  void apply(const T* u, T* f, int32_t B, cudaStream_t s, bool init = true) {
    const bool split = overlap && !halo.nbr.empty() && op->group_split < op->n_elems;
    ebe_apply_part(*op, u, f, B, s, 0, init);  // masked identity (unless written by the caller) + boundary elements
    if (!split) {
      ebe_apply_part(*op, u, f, B, s, 1, false);
      halo.run<T>(f, 3 * B, B, mask, *comm, s);
      return;
    }
    if (!side) {
      TS_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      TS_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
      TS_CUDA(cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming));
    }
    // interface rows are final after the boundary sweep: exchange them on the
    // side stream while the interior elements (which touch no interface node) run
    TS_CUDA(cudaEventRecord(ev_b, s));
    TS_CUDA(cudaStreamWaitEvent(side, ev_b, 0));
    halo.run<T>(f, 3 * B, B, mask, *comm, side);
    TS_CUDA(cudaEventRecord(ev_h, side));
    ebe_apply_part(*op, u, f, B, s, 1, false);
    TS_CUDA(cudaStreamWaitEvent(s, ev_h, 0));
  }
};

// The level-0 product with the inner PCG's (p, Ap) partials (ebe_pair_apply_dots): elements are
// partitioned, so each rank's element sums are its share; the constrained dofs' p.p counts owned
// nodes only. Same launch / exchange order as DistEbe::apply (init written by the caller).
int dist_l0_apply_dots(DistEbe& D, const float* u, float* f, int32_t B, cudaStream_t s, double* dpart,
                       const int32_t* masked_owned, int32_t n_masked_owned) {
  const bool split = D.overlap && !D.halo.nbr.empty() && D.op->group_split < D.op->n_elems;
  const int nb0 = ebe_pair_apply_dots(*D.op, u, f, B, s, dpart, 0);
  if (nb0 < 0) return -1;
  int nb1 = 0;
  if (!split) {
    nb1 = ebe_pair_apply_dots(*D.op, u, f, B, s, dpart + int64_t(nb0) * 3 * B, 1);
    D.halo.run<float>(f, 3 * B, B, D.mask, *D.comm, s);
  } else {
    if (!D.side) {
      TS_CUDA(cudaStreamCreateWithFlags(&D.side, cudaStreamNonBlocking));
      TS_CUDA(cudaEventCreateWithFlags(&D.ev_b, cudaEventDisableTiming));
      TS_CUDA(cudaEventCreateWithFlags(&D.ev_h, cudaEventDisableTiming));
    }
    TS_CUDA(cudaEventRecord(D.ev_b, s));
    TS_CUDA(cudaStreamWaitEvent(D.side, D.ev_b, 0));
    D.halo.run<float>(f, 3 * B, B, D.mask, *D.comm, D.side);
    TS_CUDA(cudaEventRecord(D.ev_h, D.side));
    nb1 = ebe_pair_apply_dots(*D.op, u, f, B, s, dpart + int64_t(nb0) * 3 * B, 1);
    TS_CUDA(cudaStreamWaitEvent(s, D.ev_h, 0));
  }
  const int used = nb0 + nb1;
  return used + ebe_masked_pp(masked_owned, n_masked_owned, u, B, s, dpart + int64_t(used) * 3 * B,
                              kRedBlocks - used);
}

struct DistVecs {
  int32_t batch = 0;
  DevBuf<double> r, q, z, p, scratch, f, u;
  DevBuf<float> r0, u0, e0, p0, q0, r1, u1, e1, p1, q1, r2, u2, e2, p2, q2;
  DevBuf<float> r2d, u2d, e2d, p2d, q2d;  // distributed level 2: owned rows (+ halo rows for u, p)
};

// Distributed level 2: this rank's coarse rows of the Galerkin operator and the
// gather halo its SpMV needs (owner values of the columns it references).
struct Level2Dist {
  int32_t n_own = 0, n_halo = 0;
  DevBuf<int32_t> own;                 // [n_own] global coarse ids, ascending
  DevBuf<int32_t> row_ptr, col_idx;    // owned rows; columns: owned [0, n_own), then halo
  DevBuf<float> blocks, m2;
  std::vector<int> nbr;                // neighbour ranks, ascending (symmetric: A2 is)
  std::vector<int64_t> soff, roff;     // [nn + 1] send / receive row offsets per neighbour
  DevBuf<int32_t> send;                // owned local ids sent, neighbour-major
  DevBuf<float> sbuf;
  // x (device, n_own + n_halo rows of width W): owner values into the halo rows
  void exchange(float* x, int W, Comm& comm, cudaStream_t s) {
    if (nbr.empty()) return;
    const int64_t ns = soff.back();
    sbuf.ensure(size_t(ns) * W);
    if (ns > 0) {
      k_halo_pack<float><<<grid_for(ns * W, 256), 256, 0, s>>>(x, send.get(), ns, W, sbuf.get());
      TS_CUDA_LAUNCH();
    }
    const int nn = static_cast<int>(nbr.size());
    std::vector<void*> sp(nn), rp(nn);
    std::vector<size_t> sb(nn), rb(nn);
    for (int k = 0; k < nn; ++k) {
      sp[k] = sbuf.get() + size_t(soff[k]) * W;
      sb[k] = size_t(soff[k + 1] - soff[k]) * W * sizeof(float);
      rp[k] = x + (size_t(n_own) + size_t(roff[k])) * W;
      rb[k] = size_t(roff[k + 1] - roff[k]) * W * sizeof(float);
    }
    comm.exchange(nn, nbr.data(), sp.data(), sb.data(), rp.data(), rb.data(), s);
  }
};

}  // namespace
}  // namespace tsg

struct ts_dist_levels {
  tsg::DistPlan plan;
  tsg::Comm* comm = nullptr;
  int32_t n0 = 0, n1 = 0, n2 = 0;
  tsg::DistEbe outer, l0, l1;
  tsg::DevBuf<int32_t> p1_ends, p1t_ptr, p1t_idx, agg, p2t_ptr, p2t_idx;
  tsg::DevBuf<int32_t> l2_row_ptr, l2_col_idx;
  tsg::DevBuf<float> l2_blocks, m0, m1, m2;
  tsg::DevBuf<uint8_t> mask0, mask1, mask2, owned0;
  tsg::DevBuf<int32_t> masked0_owned;  // constrained level-0 dofs of owned nodes (the fused gamma's p.p term)
  int32_t n_masked0_owned = 0;
  tsg::DevBuf<uint8_t> l1_dot_rows;    // level-1 rows the fused product's dots count: owned, not interface
  tsg::DevBuf<int32_t> l1_iface_owned; // owned interface rows: their dots after the exchange
  int32_t n_l1_iface_owned = 0;
  tsg::DistVecs v;
  bool l2_dist = false;  // TSGPU_DIST_L2=distributed: level 2 split by coarse rows (else replicated)
  // level 1 as this partition's assembled K1 (fp32 blocks from its own elements; interface rows then
  // summed by the level-1 halo exchange), like the single-device hierarchy; TSGPU_L1=ebe keeps the
  // element-by-element tet4 operator
  bool l1_assembled = true;
  tsg::DevBuf<int32_t> l1a_row_ptr, l1a_col_idx;
  tsg::DevBuf<float> l1a_blocks;
  tsg::DevBuf<int32_t> l1a_iface, l1a_inner;  // rows of interface vertices / the rest (overlap split)
  int32_t n_l1_iface = 0, n_l1_inner = 0;
  tsg::Level2Dist l2d;
  tsg::ColScalars cs;
  tsg::Workspace ws;
  double setup_s = 0.0;
};

namespace tsg {
namespace {

void dist_ensure_vecs(ts_dist_levels& L, int32_t B) {
  DistVecs& v = L.v;
  if (v.batch == B) return;
  const size_t l0 = 3 * size_t(L.n0) * B, l1 = 3 * size_t(L.n1) * B, l2 = 3 * size_t(L.n2) * B;
  for (auto* b : {&v.r, &v.q, &v.z, &v.p, &v.scratch}) b->alloc(l0);
  for (auto* b : {&v.r0, &v.u0, &v.e0, &v.p0, &v.q0}) b->alloc(l0);
  for (auto* b : {&v.r1, &v.u1, &v.e1, &v.p1, &v.q1}) b->alloc(l1);
  for (auto* b : {&v.r2, &v.u2, &v.e2, &v.p2, &v.q2}) b->alloc(l2);
  if (L.l2_dist) {
    const size_t own = 3 * size_t(L.l2d.n_own) * B, ext = 3 * size_t(L.l2d.n_own + L.l2d.n_halo) * B;
    for (auto* b : {&v.r2d, &v.e2d, &v.q2d}) b->alloc(std::max<size_t>(own, 1));
    for (auto* b : {&v.u2d, &v.p2d}) b->alloc(std::max<size_t>(ext, 1));
  }
  v.f.release();
  v.u.release();
  v.batch = B;
  L.cs.ensure(B);
  L.ws.ensure(B);
}

// level-1 product of a partition: assembled rows + interface sums, or the element sweep
void dist_l1_apply(ts_dist_levels& L, const float* x, float* y, int32_t B, cudaStream_t s, bool init) {
  if (L.l1_assembled) {
    DistEbe& D = L.l1;  // its halo, side stream and events
    // the staged whole-range product beats the interface-first split (two unstaged row-list
    // launches) by more than the exchange it no longer hides (TSGPU_DIST_L1_SPLIT=1 keeps the split)
    static const bool split = [] {
      const char* e = std::getenv("TSGPU_DIST_L1_SPLIT");
      return e && e[0] == '1';
    }();
    if (!D.overlap || D.halo.nbr.empty() || (!split && bcsr_rows_staged_ok(B))) {
      bcsr_rows_f32(L.l1a_row_ptr.get(), L.l1a_col_idx.get(), L.l1a_blocks.get(), L.n1, x, y, B, s, nullptr,
                    static_cast<int64_t>(L.l1a_col_idx.size()));
      D.halo.run<float>(y, 3 * B, B, L.mask1.get(), *L.comm, s);
      return;
    }
    // interface rows first; their partial sums travel while the interior rows are computed
    bcsr_rows_f32(L.l1a_row_ptr.get(), L.l1a_col_idx.get(), L.l1a_blocks.get(), L.n_l1_iface, x, y, B, s,
                  L.l1a_iface.get());
    if (!D.side) {
      TS_CUDA(cudaStreamCreateWithFlags(&D.side, cudaStreamNonBlocking));
      TS_CUDA(cudaEventCreateWithFlags(&D.ev_b, cudaEventDisableTiming));
      TS_CUDA(cudaEventCreateWithFlags(&D.ev_h, cudaEventDisableTiming));
    }
    TS_CUDA(cudaEventRecord(D.ev_b, s));
    TS_CUDA(cudaStreamWaitEvent(D.side, D.ev_b, 0));
    D.halo.run<float>(y, 3 * B, B, L.mask1.get(), *L.comm, D.side);
    TS_CUDA(cudaEventRecord(D.ev_h, D.side));
    bcsr_rows_f32(L.l1a_row_ptr.get(), L.l1a_col_idx.get(), L.l1a_blocks.get(), L.n_l1_inner, x, y, B, s,
                  L.l1a_inner.get());
    TS_CUDA(cudaStreamWaitEvent(s, D.ev_h, 0));
  } else {
    L.l1.apply<float>(x, y, B, s, init);
  }
}

// apply_multigrid_preconditioner (adaptive_cg.hpp:80-120) on a partition
void dist_mg_precond(ts_dist_levels& L, const ts_solver_config& cfg, const double* r, double* z, int32_t B,
                     ts_solve_report& rep, cudaStream_t s) {
  NvtxRange nv("dist mg preconditioner");
  DistVecs& v = L.v;
  Comm& comm = *L.comm;
  const int64_t len0 = 3 * int64_t(L.n0) * B;
  cast_d2f(r, v.r0.get(), len0, s);
  bj_apply<float>(L.m0.get(), v.r0.get(), v.u0.get(), L.n0, B, s);
  // P1^T over owned fine nodes, then sum interface vertices across ranks
  p1_restrict(v.r0.get(), v.r1.get(), L.p1t_ptr.get(), L.p1t_idx.get(), L.n1, L.mask1.get(), B, s, L.owned0.get());
  L.l1.halo.run<float>(v.r1.get(), 3 * B, B, L.mask1.get(), comm, s);
  p1_restrict(v.u0.get(), v.u1.get(), L.p1t_ptr.get(), L.p1t_idx.get(), L.n1, L.mask1.get(), B, s, L.owned0.get());
  L.l1.halo.run<float>(v.u1.get(), 3 * B, B, L.mask1.get(), comm, s);
  // P2^T over owned vertices into the (replicated) global coarse vectors
  p2_restrict(v.r1.get(), v.r2.get(), L.p2t_ptr.get(), L.p2t_idx.get(), L.n2, L.mask2.get(), B, s);
  comm.allreduce_sum(v.r2.get(), 3 * size_t(L.n2) * B, s);
  p2_restrict(v.u1.get(), v.u2.get(), L.p2t_ptr.get(), L.p2t_idx.get(), L.n2, L.mask2.get(), B, s);
  comm.allreduce_sum(v.u2.get(), 3 * size_t(L.n2) * B, s);
  const auto t0 = clk::now();
  InnerStats s2;
  if (L.l2_dist) {  // this rank's coarse rows; halo exchange in every product, all-reduced dots
    Level2Dist& D = L.l2d;
    const int W = 3 * B;
    if (D.n_own > 0) {
      k_gather_rows<float><<<grid_for(int64_t(D.n_own) * W, 256), 256, 0, s>>>(v.r2.get(), D.own.get(), D.n_own, W,
                                                                               v.r2d.get());
      TS_CUDA_LAUNCH();
      k_gather_rows<float><<<grid_for(int64_t(D.n_own) * W, 256), 256, 0, s>>>(v.u2.get(), D.own.get(), D.n_own, W,
                                                                               v.u2d.get());
      TS_CUDA_LAUNCH();
    }
    L.ws.comm = L.comm;
    L.ws.owned = nullptr;
    auto a2 = [&](const float* x, float* y, bool) {
      D.exchange(const_cast<float*>(x), W, comm, s);
      bcsr_apply_f32(D.row_ptr.get(), D.col_idx.get(), D.blocks.get(), D.n_own, x, y, B, s,
                     static_cast<int64_t>(D.col_idx.size()));
    };
    s2 = inner_pcg<float>(a2, D.m2.get(), v.r2d.get(), v.u2d.get(), D.n_own, B, cfg.level_tol[2],
                          cfg.level_max_iter[2], v.e2d.get(), v.p2d.get(), v.q2d.get(), L.cs, L.ws, s);
    TS_CUDA(cudaMemsetAsync(v.u2.get(), 0, 3 * size_t(L.n2) * B * sizeof(float), s));
    if (D.n_own > 0) {
      k_scatter_rows<float><<<grid_for(int64_t(D.n_own) * W, 256), 256, 0, s>>>(v.u2d.get(), D.own.get(), D.n_own,
                                                                                W, v.u2.get());
      TS_CUDA_LAUNCH();
    }
    comm.allreduce_sum(v.u2.get(), 3 * size_t(L.n2) * B, s);  // every rank: the whole coarse correction
  } else {
    L.ws.comm = nullptr;  // level 2 is replicated: identical on every rank, no collectives
    L.ws.owned = nullptr;
    auto a2 = [&](const float* x, float* y, bool) {
      bcsr_apply_f32(L.l2_row_ptr.get(), L.l2_col_idx.get(), L.l2_blocks.get(), L.n2, x, y, B, s,
                     static_cast<int64_t>(L.l2_col_idx.size()));
    };
    const std::function<int(const float*, float*)> a2_dots = [&](const float* x, float* y) {
      return bcsr_apply_f32_gamma(L.l2_row_ptr.get(), L.l2_col_idx.get(), L.l2_blocks.get(), L.n2, x, y, B, s,
                                  static_cast<int64_t>(L.l2_col_idx.size()), L.ws)
                 ? 1 : 0;
    };
    s2 = inner_pcg<float>(a2, L.m2.get(), v.r2.get(), v.u2.get(), L.n2, B, cfg.level_tol[2], cfg.level_max_iter[2],
                          v.e2.get(), v.p2.get(), v.q2.get(), L.cs, L.ws, s, false, nullptr, &a2_dots);
  }
  const auto t1 = clk::now();
  L.ws.comm = L.comm;
  L.ws.owned = L.owned0.get();  // the vertex prefix of the level-0 flags
  p2_apply(v.u2.get(), v.u1.get(), L.agg.get(), L.n1, L.mask1.get(), B, s);
  auto a1 = [&](const float* x, float* y, bool init) { dist_l1_apply(L, x, y, B, s, init); };
  // the staged whole-range product (dist_l1_apply's unsplit form) with gamma's dots of this rank's
  // owned rows: interior ones in the product, interface ones after the exchange completes them
  const std::function<int(const float*, float*)> a1_dots = [&](const float* x, float* y) {
    static const bool split = [] {
      const char* e = std::getenv("TSGPU_DIST_L1_SPLIT");
      return e && e[0] == '1';
    }();
    if (!L.l1_assembled || split) return 0;
    if (!bcsr_rows_f32_gamma(L.l1a_row_ptr.get(), L.l1a_col_idx.get(), L.l1a_blocks.get(), L.n1, x, y, B, s,
                             static_cast<int64_t>(L.l1a_col_idx.size()), L.ws, L.l1_dot_rows.get()))
      return 0;
    L.l1.halo.run<float>(y, 3 * B, B, L.mask1.get(), *L.comm, s);
    rows_dots_append(x, y, L.l1_iface_owned.get(), L.n_l1_iface_owned, B, s, L.ws);
    return 1;
  };
  const InnerStats s1 = inner_pcg<float>(a1, L.m1.get(), v.r1.get(), v.u1.get(), L.n1, B, cfg.level_tol[1],
                                         cfg.level_max_iter[1], v.e1.get(), v.p1.get(), v.q1.get(), L.cs, L.ws, s,
                                         !L.l1_assembled, L.mask1.get(), &a1_dots);
  const auto t2 = clk::now();
  p1_apply(v.u1.get(), v.u0.get(), L.p1_ends.get(), L.n1, L.n0, L.mask0.get(), B, s);
  auto a0 = [&](const float* x, float* y, bool init) { L.l0.apply<float>(x, y, B, s, init); };
  const std::function<int(const float*, float*)> a0_dots = [&](const float* x, float* y) {
    L.ws.ensure(B);
    const int nb = dist_l0_apply_dots(L.l0, x, y, B, s, L.ws.partial.get(), L.masked0_owned.get(),
                                      L.n_masked0_owned);
    if (nb < 0) return 0;
    L.ws.nblk = nb;
    return 2;
  };
  const InnerStats s0 = inner_pcg<float>(a0, L.m0.get(), v.r0.get(), v.u0.get(), L.n0, B, cfg.level_tol[0],
                                         cfg.level_max_iter[0], v.e0.get(), v.p0.get(), v.q0.get(), L.cs, L.ws, s,
                                         true, L.mask0.get(), &a0_dots);
  const auto t3 = clk::now();
  rep.inner_iterations[2] += s2.iterations;
  rep.inner_iterations[1] += s1.iterations;
  rep.inner_iterations[0] += s0.iterations;
  rep.time_inner_s[2] += secs(t0, t1);
  rep.time_inner_s[1] += secs(t1, t2);
  rep.time_inner_s[0] += secs(t2, t3);
  cast_f2d(v.u0.get(), z, len0, s);
}

std::vector<double> per_element(const Mesh& m, int32_t n_mat, const double* x) {
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

// The distributed level 2 of one rank, from the replicated global operator every rank
// holds after the broadcast: coarse row a belongs to the owner of its lowest vertex
// (a vertex's owner is the lowest rank touching it), so a rank's coarse rows sit on its
// partition; its SpMV needs the owner values of the off-rank columns it references.
void build_level2_dist(ts_dist_levels& L, const Mesh& m, const int32_t* part, const std::vector<int32_t>& agg_g,
                       const std::vector<int32_t>& rp2, const std::vector<int32_t>& ci2, const std::vector<float>& bl2,
                       const std::vector<float>& m2h) {
  const int me = L.comm->rank(), P = L.comm->size();
  const int32_t V = m.vertex_count, n2 = L.n2;
  std::vector<int32_t> vown(V, INT32_MAX), owner(n2, -1);
  for (int32_t e = 0; e < m.n_elems(); ++e)
    for (int a = 0; a < 4; ++a) {
      int32_t& o = vown[m.tets10[10 * size_t(e) + a]];
      o = std::min(o, part[e]);
    }
  for (int32_t v = 0; v < V; ++v)  // ascending: the aggregate's lowest vertex decides
    if (owner[agg_g[v]] < 0) owner[agg_g[v]] = vown[v] == INT32_MAX ? 0 : vown[v];
  Level2Dist& D = L.l2d;
  std::vector<int32_t> own, loc(n2, -1);
  for (int32_t a = 0; a < n2; ++a)
    if (owner[a] == me) {
      loc[a] = static_cast<int32_t>(own.size());
      own.push_back(a);
    }
  D.n_own = static_cast<int32_t>(own.size());
  // halo: off-rank columns of my rows, by owner rank then global id
  std::vector<std::vector<int32_t>> need(P);
  {
    std::vector<uint8_t> seen(n2, 0);
    for (int32_t a : own)
      for (int32_t q = rp2[a]; q < rp2[a + 1]; ++q) {
        const int32_t c = ci2[q];
        if (owner[c] != me && !seen[c]) {
          seen[c] = 1;
          need[owner[c]].push_back(c);
        }
      }
  }
  D.roff.assign(1, 0);
  D.nbr.clear();
  for (int k = 0; k < P; ++k) {
    if (need[k].empty()) continue;
    std::sort(need[k].begin(), need[k].end());
    for (size_t i = 0; i < need[k].size(); ++i)
      loc[need[k][i]] = D.n_own + static_cast<int32_t>(D.roff.back() + static_cast<int64_t>(i));
    D.nbr.push_back(k);
    D.roff.push_back(D.roff.back() + static_cast<int64_t>(need[k].size()));
  }
  D.n_halo = static_cast<int32_t>(D.roff.back());
  // what each neighbour needs from me: my coarse rows referenced by its rows (same order it expects)
  std::vector<int32_t> send;
  D.soff.assign(1, 0);
  for (int k : D.nbr) {
    std::vector<int32_t> want;
    std::vector<uint8_t> seen(n2, 0);
    for (int32_t a = 0; a < n2; ++a) {
      if (owner[a] != k) continue;
      for (int32_t q = rp2[a]; q < rp2[a + 1]; ++q) {
        const int32_t c = ci2[q];
        if (owner[c] == me && !seen[c]) {
          seen[c] = 1;
          want.push_back(c);
        }
      }
    }
    std::sort(want.begin(), want.end());
    for (int32_t c : want) send.push_back(loc[c]);
    D.soff.push_back(static_cast<int64_t>(send.size()));
  }
  // my rows with local column ids, their block-Jacobi blocks
  std::vector<int32_t> rp(1, 0), ci;
  std::vector<float> bl, mb;
  for (int32_t a : own) {
    for (int32_t q = rp2[a]; q < rp2[a + 1]; ++q) {
      ci.push_back(loc[ci2[q]]);
      bl.insert(bl.end(), bl2.begin() + 9 * size_t(q), bl2.begin() + 9 * size_t(q + 1));
    }
    rp.push_back(static_cast<int32_t>(ci.size()));
    mb.insert(mb.end(), m2h.begin() + 9 * size_t(a), m2h.begin() + 9 * size_t(a + 1));
  }
  D.own.upload(own);
  D.row_ptr.upload(rp);
  D.col_idx.upload(ci);
  D.blocks.upload(bl);
  D.m2.upload(mb);
  D.send.upload(send);
}

}  // namespace

// build_solver_levels (adaptive_cg.hpp:39-67) for one partition
ts_dist_levels* dist_levels_create(const Mesh& m, int32_t n_mat, const double* lam, const double* mu,
                                   const uint8_t* dof_mask, const int32_t* part, const ts_solver_config& cfg,
                                   Comm* comm) {
  const auto t0 = clk::now();
  if (ts_config_validate(&cfg) != TS_OK) fail(TS_ERR_VALIDATION, ts_last_error());
  if (!comm) validation("dist levels: communicator required");
  require_device();
  TS_CUDA(cudaSetDevice(comm->device()));
  auto L = std::make_unique<ts_dist_levels>();
  L->comm = comm;
  const std::vector<uint8_t> gmask = dof_mask ? std::vector<uint8_t>(dof_mask, dof_mask + 3 * size_t(m.n_nodes()))
                                              : m.dirichlet_mask();
  L->plan = build_dist_plan(m, gmask.data(), part, comm->size(), comm->rank());
  const DistPlan& P = L->plan;
  L->n0 = P.n_local;
  L->n1 = P.n_local_vertices;
  std::vector<uint8_t> group(P.elems.size());
  for (size_t k = 0; k < group.size(); ++k) group[k] = P.elem_boundary[k] ? 0 : 1;
  const std::vector<uint8_t> mask1(P.mask.begin(), P.mask.begin() + 3 * size_t(L->n1));
  L->outer.op.reset(ebe_create(P.local, 2, n_mat, lam, mu, P.mask.data(), 64, group.data()));
  L->l0.op.reset(ebe_create(P.local, 2, n_mat, lam, mu, P.mask.data(), 32, group.data()));
  L->l1.op.reset(ebe_create(P.local, 1, n_mat, lam, mu, mask1.data(), 32, group.data()));
  L->mask0.upload(P.mask);
  L->mask1.upload(mask1);
  L->owned0.upload(P.owned);
  {
    std::vector<int32_t> mo;
    for (size_t d = 0; d < P.mask.size(); ++d)
      if (P.mask[d] && P.owned[d / 3]) mo.push_back(static_cast<int32_t>(d));
    L->n_masked0_owned = static_cast<int32_t>(mo.size());
    L->masked0_owned.upload(mo);
  }
  for (DistEbe* d : {&L->outer, &L->l0}) {
    d->halo.build(P.halo0);
    d->mask = L->mask0.get();
    d->comm = comm;
  }
  L->l1.halo.build(P.halo1);
  L->l1.mask = L->mask1.get();
  L->l1.comm = comm;
  if (const char* e = std::getenv("TSGPU_DIST_OVERLAP"))
    for (DistEbe* d : {&L->outer, &L->l0, &L->l1}) d->overlap = e[0] != '0';
  // geometric P1 on the partition; transpose over OWNED fine nodes only, so
  // the per-rank restrictions sum to the global one after the vertex exchange
  {
    const Mesh& lm = P.local;
    const int32_t N = L->n0, V = L->n1;
    static constexpr int ee[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
    std::vector<int32_t> ends(2 * size_t(N - V), -1);
    for (int32_t e = 0; e < lm.n_elems(); ++e) {
      const int32_t* t = lm.tets10.data() + 10 * size_t(e);
      for (int q = 0; q < 6; ++q) {
        int32_t a = t[ee[q][0]], b = t[ee[q][1]];
        if (a > b) std::swap(a, b);
        const int32_t mid = t[4 + q];
        if (mid < V || a >= V || b >= V) validation("dist P1: vertex / edge numbering broken");
        ends[2 * size_t(mid - V)] = a;
        ends[2 * size_t(mid - V) + 1] = b;
      }
    }
    std::vector<int32_t> tptr(V + 1, 0);
    auto owned = [&](int32_t i) { return P.owned[i] != 0; };
    for (int32_t k = 0; k < N - V; ++k) {
      if (ends[2 * size_t(k)] < 0) validation("dist P1: edge node without endpoints");
      if (!owned(k + V)) continue;
      ++tptr[ends[2 * size_t(k)] + 1];
      ++tptr[ends[2 * size_t(k) + 1] + 1];
    }
    for (int32_t i = 0; i < V; ++i) tptr[i + 1] += tptr[i];
    std::vector<int32_t> tidx(tptr[V]), cur(tptr.begin(), tptr.end() - 1);
    for (int32_t k = 0; k < N - V; ++k) {
      if (!owned(k + V)) continue;
      tidx[cur[ends[2 * size_t(k)]]++] = k + V;
      tidx[cur[ends[2 * size_t(k) + 1]]++] = k + V;
    }
    L->p1_ends.upload(ends);
    L->p1t_ptr.upload(tptr);
    L->p1t_idx.upload(tidx);
  }
  // level 2: the reference's sequential aggregation of the GLOBAL K1 (identical to the
  // single-device hierarchy), built ONCE on rank 0 with all host cores and broadcast
  {
    const int32_t V = m.vertex_count;
    int64_t sizes[2] = {0, 0};  // n2, nnzb2
    std::vector<int32_t> agg_g(V), rp2, ci2;
    std::vector<float> bl2, m2h;
    std::vector<uint8_t> mk2;
    if (comm->rank() == 0) {
      const int saved = omp_get_max_threads();
      omp_set_num_threads(omp_get_num_procs());
      const std::vector<uint8_t> gmask1(gmask.begin(), gmask.begin() + 3 * size_t(V));
      Level2Host l2 = build_level2_host(m, per_element(m, n_mat, lam), per_element(m, n_mat, mu), gmask1,
                                        cfg.aggregate_target);
      omp_set_num_threads(saved);
      sizes[0] = l2.n2;
      sizes[1] = l2.row_ptr[l2.n2];
      agg_g = std::move(l2.agg_of_node);
      rp2 = std::move(l2.row_ptr);
      ci2 = std::move(l2.col_idx);
      bl2 = std::move(l2.blocks);
      m2h = std::move(l2.m2);
      mk2 = std::move(l2.mask2);
    }
    comm->broadcast(sizes, sizeof sizes, 0);
    L->n2 = static_cast<int32_t>(sizes[0]);
    rp2.resize(size_t(L->n2) + 1);
    ci2.resize(sizes[1]);
    bl2.resize(9 * size_t(sizes[1]));
    m2h.resize(9 * size_t(L->n2));
    mk2.resize(3 * size_t(L->n2));
    comm->broadcast(agg_g.data(), agg_g.size() * sizeof(int32_t), 0);
    comm->broadcast(rp2.data(), rp2.size() * sizeof(int32_t), 0);
    comm->broadcast(ci2.data(), ci2.size() * sizeof(int32_t), 0);
    comm->broadcast(bl2.data(), bl2.size() * sizeof(float), 0);
    comm->broadcast(m2h.data(), m2h.size() * sizeof(float), 0);
    comm->broadcast(mk2.data(), mk2.size(), 0);
    L->l2_row_ptr.upload(rp2);
    L->l2_col_idx.upload(ci2);
    L->l2_blocks.upload(bl2);
    L->m2.upload(m2h);
    L->mask2.upload(mk2);
    // level 2 replicated on every rank (no collectives inside its PCG, but every rank does all of
    // it) or split by coarse rows (1/P of it, plus a gather halo per product and all-reduced dots);
    // TSGPU_DIST_L2 = replicated | distributed | auto (default: split from 4 ranks on, where the
    // replicated coarse solve becomes the Amdahl term — DESIGN.md §6)
    {
      const char* e = std::getenv("TSGPU_DIST_L2");
      const std::string mode = e ? e : "auto";
      L->l2_dist = mode == "distributed" || (mode == "auto" && comm->size() >= 4);
    }
    if (L->l2_dist) build_level2_dist(*L, m, part, agg_g, rp2, ci2, bl2, m2h);
    const int32_t Vl = L->n1;
    std::vector<int32_t> agg_l(Vl), aptr(L->n2 + 1, 0);
    for (int32_t i = 0; i < Vl; ++i) {
      agg_l[i] = agg_g[P.l2g[i]];
      if (P.owned[i]) ++aptr[agg_l[i] + 1];
    }
    for (int32_t a = 0; a < L->n2; ++a) aptr[a + 1] += aptr[a];
    std::vector<int32_t> amem(aptr[L->n2]), cur(aptr.begin(), aptr.end() - 1);
    for (int32_t i = 0; i < Vl; ++i)  // ascending local = ascending global vertex id
      if (P.owned[i]) amem[cur[agg_l[i]]++] = i;
    L->agg.upload(agg_l);
    L->p2t_ptr.upload(aptr);
    L->p2t_idx.upload(amem);
  }
  // block Jacobi: interface diagonal blocks summed across ranks, then inverted
  {
    cudaStream_t s = nullptr;
    L->m0.alloc(9 * size_t(L->n0));
    L->m1.alloc(9 * size_t(L->n1));
    DevBuf<double> d0(9 * size_t(L->n0)), d1(9 * size_t(L->n1));
    ebe_diag_blocks(*L->l0.op, d0.get(), s);
    ebe_diag_blocks(*L->l1.op, d1.get(), s);
    L->l0.halo.run<double>(d0.get(), 9, 3, nullptr, *comm, s);
    L->l1.halo.run<double>(d1.get(), 9, 3, nullptr, *comm, s);
    bj_invert(d0.get(), L->mask0.get(), L->n0, 32, L->m0.get(), s);
    bj_invert(d1.get(), L->mask1.get(), L->n1, 32, L->m1.get(), s);
    for (ts_ebe* op : {L->l0.op.get(), L->l1.op.get(), L->outer.op.get()}) HostVec<double>().swap(op->coef64);
  }
  if (const char* e = std::getenv("TSGPU_L1")) L->l1_assembled = std::string(e) != "ebe";
  if (L->l1_assembled) {  // this partition's K1 (float-rounded inputs, ebe_operator.hpp:54-62)
    HostVec<float> k1f;
    const BcsrD k1 = assemble_tet4(P.local, per_element(P.local, n_mat, lam), per_element(P.local, n_mat, mu), mask1,
                                   &k1f);
    L->l1a_row_ptr.upload(k1.row_ptr);
    L->l1a_col_idx.upload(k1.col_idx);
    L->l1a_blocks.upload(k1f);
    {  // rows of the level-1 interface vertices (exchanged) and the rest (computed under the exchange)
      std::vector<uint8_t> iface(L->n1, 0);
      for (int32_t v : P.halo1.sh_nodes) iface[v] = 1;
      std::vector<int32_t> ri, rn;
      for (int32_t v = 0; v < L->n1; ++v) (iface[v] ? ri : rn).push_back(v);
      L->n_l1_iface = static_cast<int32_t>(ri.size());
      L->n_l1_inner = static_cast<int32_t>(rn.size());
      std::vector<uint8_t> sel(L->n1, 0);
      std::vector<int32_t> io;
      for (int32_t v = 0; v < L->n1; ++v) {
        if (!P.owned[v]) continue;
        if (iface[v]) io.push_back(v);
        else sel[v] = 1;
      }
      L->l1_dot_rows.upload(sel);
      L->l1_iface_owned.upload(io);
      L->n_l1_iface_owned = static_cast<int32_t>(io.size());
      L->l1a_iface.upload(ri);
      L->l1a_inner.upload(rn);
    }
    TS_CUDA(cudaDeviceSynchronize());
    L->l1.op.reset();  // the element operator only served the block-Jacobi diagonal
  }
  TS_CUDA(cudaDeviceSynchronize());
  comm->barrier();
  L->setup_s = secs(t0, clk::now());
  return L.release();
}

// solve (adaptive_cg.hpp:242-263) on this rank's partition (device buffers in local node order)
void dist_solve_device(ts_dist_levels& L, const double* f, const double* u0, double* u, int32_t B,
                       const ts_solver_config& cfg, ts_solve_report& rep, cudaStream_t s) {
  if (ts_config_validate(&cfg) != TS_OK) fail(TS_ERR_VALIDATION, ts_last_error());
  if (B < 1 || B > kRedThreads) validation("solve: batch must be in [1, 256]");
  TS_CUDA(cudaSetDevice(L.comm->device()));
  dist_ensure_vecs(L, B);
  L.ws.comm = L.comm;
  L.ws.owned = L.owned0.get();
  dot2<double>(f, f, nullptr, nullptr, 3 * int64_t(L.n0), B, L.cs[ColScalars::FN2], L.ws, s);
  std::vector<double> fn2(B);
  TS_CUDA(cudaMemcpyAsync(fn2.data(), L.cs[ColScalars::FN2], B * sizeof(double), cudaMemcpyDeviceToHost, s));
  TS_CUDA(cudaStreamSynchronize(s));
  bool any = false;
  for (double x : fn2) any |= x != 0.0;
  if (!any) validation("solve: right-hand side has no nonzero column");
  report_reset(rep, 0, 32);
  rep.time_setup_s = L.setup_s;
  if (u != u0) TS_CUDA(cudaMemcpyAsync(u, u0, 3 * size_t(L.n0) * B * sizeof(double), cudaMemcpyDeviceToDevice, s));
  auto precond = [&](const double* r, double* z) {
    dist_mg_precond(L, cfg, r, z, B, rep, s);
    L.ws.comm = L.comm;
    L.ws.owned = L.owned0.get();
  };
  auto kop = [&](const double* x, double* y) { L.outer.apply<double>(x, y, B, s); };
  run_outer_cg(kop, L.n0, f, u, B, cfg.outer_tol, cfg.outer_max_iter, cfg.residual_history_stride, precond, L.v,
               L.cs, L.ws, rep, s);
}

void dist_ebe_apply(ts_dist_levels& L, int which, const void* u, void* f, int32_t B, cudaStream_t s) {
  TS_CUDA(cudaSetDevice(L.comm->device()));
  if (which == 0) L.outer.apply<double>(static_cast<const double*>(u), static_cast<double*>(f), B, s);
  else if (which == 1) L.l0.apply<float>(static_cast<const float*>(u), static_cast<float*>(f), B, s);
  else if (which == 2) dist_l1_apply(L, static_cast<const float*>(u), static_cast<float*>(f), B, s, true);
  else validation("dist apply: operator must be 0 (outer), 1 (level 0) or 2 (level 1)");
}

void dist_levels_destroy(ts_dist_levels* L) { delete L; }

void dist_levels_sizes(const ts_dist_levels& L, int32_t* n0, int32_t* n1, int32_t* n2) {
  if (n0) *n0 = L.n0;
  if (n1) *n1 = L.n1;
  if (n2) *n2 = L.n2;
}

const std::vector<int32_t>& dist_local_nodes(const ts_dist_levels& L) { return L.plan.l2g; }

void dist_levels_info(const ts_dist_levels& L, int32_t* n_elements, int64_t* halo_rows0, int32_t* n_nbr,
                      double* setup_s) {
  *n_elements = static_cast<int32_t>(L.plan.elems.size());
  *halo_rows0 = L.plan.halo0.rows_total();
  *n_nbr = static_cast<int32_t>(L.plan.halo0.nbr.size());
  *setup_s = L.setup_s;
}
Comm* dist_levels_comm(const ts_dist_levels& L) { return L.comm; }
const uint8_t* dist_levels_mask0(const ts_dist_levels& L) { return L.mask0.get(); }

// host-buffer solve: H2D of f / u0, solve on a private stream, D2H of u
void dist_solve_host(ts_dist_levels& L, const double* f, const double* u0, double* u, int32_t B,
                     const ts_solver_config& cfg, ts_solve_report& rep) {
  TS_CUDA(cudaSetDevice(L.comm->device()));
  if (B < 1 || B > kRedThreads) validation("solve: batch must be in [1, 256]");
  dist_ensure_vecs(L, B);
  const size_t len = 3 * size_t(L.n0) * B;
  DistVecs& v = L.v;
  if (!v.f.get()) {
    v.f.alloc(len);
    v.u.alloc(len);
  }
  cudaStream_t s = nullptr;
  TS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    ~Guard() { cudaStreamDestroy(s); }
  } g{s};
  TS_CUDA(cudaMemcpyAsync(v.f.get(), f, len * sizeof(double), cudaMemcpyHostToDevice, s));
  TS_CUDA(cudaMemcpyAsync(v.u.get(), u0, len * sizeof(double), cudaMemcpyHostToDevice, s));
  ts_status rc = TS_OK;
  std::string msg;
  try {
    dist_solve_device(L, v.f.get(), v.u.get(), v.u.get(), B, cfg, rep, s);
  } catch (const Error& e) {
    rc = e.code;
    msg = e.what();
  }
  if (rc == TS_OK || rc == TS_ERR_NO_CONVERGENCE) {
    TS_CUDA(cudaMemcpyAsync(u, v.u.get(), len * sizeof(double), cudaMemcpyDeviceToHost, s));
    TS_CUDA(cudaStreamSynchronize(s));
  }
  if (rc != TS_OK) fail(rc, msg);
}

// ---- a standalone partitioned EBE operator (no level hierarchy): bench / users
// that only need K u on a partitioned mesh
}  // namespace tsg

struct ts_dist_ebe {
  tsg::DistPlan plan;
  tsg::DistEbe d;
  tsg::DevBuf<uint8_t> mask;
};

namespace tsg {

ts_dist_ebe* dist_ebe_create(const Mesh& m, int order, int32_t n_mat, const double* lam, const double* mu,
                             const uint8_t* dof_mask, const int32_t* part, int prec, Comm* comm) {
  if (!comm) validation("dist ebe: communicator required");
  require_device();
  TS_CUDA(cudaSetDevice(comm->device()));
  auto D = std::make_unique<ts_dist_ebe>();
  const std::vector<uint8_t> gmask = dof_mask ? std::vector<uint8_t>(dof_mask, dof_mask + 3 * size_t(m.n_nodes()))
                                              : m.dirichlet_mask();
  D->plan = build_dist_plan(m, gmask.data(), part, comm->size(), comm->rank());
  const DistPlan& P = D->plan;
  std::vector<uint8_t> group(P.elems.size());
  for (size_t k = 0; k < group.size(); ++k) group[k] = P.elem_boundary[k] ? 0 : 1;
  const int32_t nn = order == 1 ? P.n_local_vertices : P.n_local;
  const std::vector<uint8_t> mk(P.mask.begin(), P.mask.begin() + 3 * size_t(nn));
  D->d.op.reset(ebe_create(P.local, order, n_mat, lam, mu, mk.data(), prec, group.data()));
  HostVec<double>().swap(D->d.op->coef64);
  D->mask.upload(mk);
  D->d.halo.build(order == 1 ? P.halo1 : P.halo0);
  D->d.mask = D->mask.get();
  D->d.comm = comm;
  if (const char* e = std::getenv("TSGPU_DIST_OVERLAP")) D->d.overlap = e[0] != '0';
  TS_CUDA(cudaDeviceSynchronize());
  comm->barrier();
  return D.release();
}

void dist_ebe_destroy(ts_dist_ebe* D) { delete D; }

void dist_ebe_info(const ts_dist_ebe& D, int32_t* n_local, int32_t* n_elems, int64_t* halo_rows, int32_t* n_nbr) {
  if (n_local) *n_local = D.d.op->n_nodes;
  if (n_elems) *n_elems = D.d.op->n_elems;
  if (halo_rows) *halo_rows = D.d.halo.roff.empty() ? 0 : D.d.halo.roff.back();
  if (n_nbr) *n_nbr = static_cast<int32_t>(D.d.halo.nbr.size());
}

const std::vector<int32_t>& dist_ebe_local_nodes(const ts_dist_ebe& D) { return D.plan.l2g; }

void dist_ebe_apply_op(ts_dist_ebe& D, const void* u, void* f, int32_t B, cudaStream_t s) {
  TS_CUDA(cudaSetDevice(D.d.comm->device()));
  if (D.d.op->prec == 64) D.d.apply<double>(static_cast<const double*>(u), static_cast<double*>(f), B, s);
  else D.d.apply<float>(static_cast<const float*>(u), static_cast<float*>(f), B, s);
}

ts_ebe* dist_ebe_local(ts_dist_ebe& D) { return D.d.op.get(); }
Comm* dist_ebe_comm(const ts_dist_ebe& D) { return D.d.comm; }

}  // namespace tsg
