// ebe_color.cu — the deterministic EBE sweep: greedy element coloring
// (build_coloring, ebe_operator.hpp:190-214) and one launch per color.
//
// The default sweeps scatter with L2 atomics, so the order in which a node's
// element contributions are summed depends on scheduling; results then agree
// with the reference only to rounding. The reference's contract is stronger
// (SPEC determinism; test_ebe.cpp:254-269 batched columns equal single-column
// products bit for bit, :296-317 colored path bit-identical across runs and
// worker counts, test_solver.cpp:183-201 identical columns stay identical).
// Here no two elements of a color share a node, so each color adds its
// contributions with plain read-add-writes and every node sums its elements in
// ascending color order: the bits depend only on the mesh, never on the batch
// width, the launch geometry or the run. One thread per (element, case) with
// the same non-contracting element product for every case keeps columns
// independent of the batch. Cost: ~30 launches (tet10) that each move their
// share of f through HBM — a correctness mode (the C++ drop-in's default),
// not the throughput path.
#include <algorithm>
#include <cstring>
#include <vector>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {
namespace {

template <typename T, int NPE, int CS>
__global__ void k_ebe_colored(const int32_t* __restrict__ conn3, const T* __restrict__ coef,
                              const int32_t* __restrict__ elems, int32_t ne, const T* __restrict__ u,
                              T* __restrict__ f, int32_t B) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(ne) * B) return;
  const int64_t k = t / B;
  const int b = static_cast<int>(t - k * B);
  const int64_t e = elems[k];
  const int32_t* c = conn3 + CS * e;
  const uint32_t mw = static_cast<uint32_t>(c[NPE]);
  T uu[NPE][3];
#pragma unroll
  for (int a = 0; a < NPE; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q)
      uu[a][q] = ((mw >> (3 * a + q)) & 1u) ? T(0) : u[(int64_t(c[a]) + q) * B + b];
  const T* r = coef + 12 * e;
  T bb[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int d = 0; d < 3; ++d) bb[i][d] = r[3 * i + d];
  T ff[NPE][3];
  if constexpr (NPE == 10) tet10_product<T>(uu, bb, r[9], r[10], ff);
  else tet4_product<T>(uu, bb, r[9], r[10], ff);
#pragma unroll
  for (int a = 0; a < NPE; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (!((mw >> (3 * a + q)) & 1u)) {
        T* p = f + (int64_t(c[a]) + q) * B + b;
        *p = LaneOps<T>::add(*p, ff[a][q]);
      }
}

void build_coloring(ts_ebe& op) {
  const int npe = op.npe;
  const int64_t E = op.n_elems;
  if (op.host_conn.size() != size_t(E) * npe) validation("deterministic sweep: operator setup data released");
  // first-fit over sweep positions with a per-node bitmask of used colors (<= 128 colors)
  std::vector<std::array<uint64_t, 2>> used(op.n_nodes, std::array<uint64_t, 2>{0, 0});
  std::vector<uint8_t> color(E);
  int n_colors = 0;
  for (int64_t i = 0; i < E; ++i) {
    uint64_t w0 = 0, w1 = 0;
    for (int a = 0; a < npe; ++a) {
      const auto& m = used[op.host_conn[i * npe + a]];
      w0 |= m[0];
      w1 |= m[1];
    }
    int c = 0;
    if (~w0) c = __builtin_ctzll(~w0);
    else if (~w1) c = 64 + __builtin_ctzll(~w1);
    else validation("deterministic sweep: more than 128 element colors");
    color[i] = static_cast<uint8_t>(c);
    n_colors = std::max(n_colors, c + 1);
    for (int a = 0; a < npe; ++a) used[op.host_conn[i * npe + a]][c / 64] |= uint64_t(1) << (c % 64);
  }
  auto plan = std::make_unique<EbeColorPlan>();
  plan->n_colors = n_colors;
  // one list per (element group, color): a partitioned operator sweeps its groups separately
  const int64_t split = op.group_split;
  plan->color_ptr.assign(2 * size_t(n_colors) + 1, 0);
  for (int64_t i = 0; i < E; ++i) ++plan->color_ptr[(i >= split ? n_colors : 0) + color[i] + 1];
  for (size_t k = 0; k + 1 < plan->color_ptr.size(); ++k) plan->color_ptr[k + 1] += plan->color_ptr[k];
  std::vector<int32_t> elems(E), cur(plan->color_ptr.begin(), plan->color_ptr.end() - 1);
  for (int64_t i = 0; i < E; ++i) elems[cur[(i >= split ? n_colors : 0) + color[i]]++] = static_cast<int32_t>(i);
  plan->elems.upload(elems);
  TS_CUDA(cudaDeviceSynchronize());
  op.color = std::move(plan);
}

template <typename T>
void color_apply_t(const ts_ebe& op, const T* u, T* f, int32_t B, cudaStream_t s, int part) {
  const EbeColorPlan& cp = *op.color;
  const int g0 = part == 1 ? 1 : 0, g1 = part == 0 ? 1 : 2;
  for (int g = g0; g < g1; ++g)
    for (int c = 0; c < cp.n_colors; ++c) {
      const int32_t k0 = cp.color_ptr[g * cp.n_colors + c], k1 = cp.color_ptr[g * cp.n_colors + c + 1];
      if (k1 <= k0) continue;
      const unsigned grid = grid_for(int64_t(k1 - k0) * B, 128);
      if (op.order == 2)
        k_ebe_colored<T, 10, 12><<<grid, 128, 0, s>>>(op.conn3.get(), reinterpret_cast<const T*>(op.coef.get()),
                                                      cp.elems.get() + k0, k1 - k0, u, f, B);
      else
        k_ebe_colored<T, 4, 8><<<grid, 128, 0, s>>>(op.conn3.get(), reinterpret_cast<const T*>(op.coef.get()),
                                                    cp.elems.get() + k0, k1 - k0, u, f, B);
      TS_CUDA_LAUNCH();
    }
}

}  // namespace

void ebe_set_deterministic(ts_ebe& op, bool on) {
  if (on && !op.color) build_coloring(op);
  op.deterministic = on;
}

void ebe_color_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part) {
  if (!op.color) validation("deterministic sweep: no element coloring (ebe_set_deterministic)");
  if (op.prec == 32) color_apply_t<float>(op, static_cast<const float*>(u), static_cast<float*>(f), batch, s, part);
  else color_apply_t<double>(op, static_cast<const double*>(u), static_cast<double*>(f), batch, s, part);
}

}  // namespace tsg
