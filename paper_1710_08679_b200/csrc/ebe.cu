// ebe.cu — the hot path: multi-case matrix-free EBE stiffness product on sm_100a.
//
// Replaces EbeOperator<T>::apply (ebe_operator.hpp:90-188). Layout follows the
// reference: u/f are [node][axis][case] (vector_batch.hpp:12-28), so the r
// cases of one dof are contiguous and one element sweep serves all of them
// (the paper's "dense computation").
//
// Kernel design (B200):
//  * one lane group of TPE threads per element; each thread owns CPT = 2
//    consecutive fp32 cases (one 8-byte lane vector, packed FFMA2 math) or
//    1 fp64 case; connectivity and the 12-scalar coefficient record are read
//    once per lane group (broadcast) and reused across the r cases;
//  * element data are the gradient/material coefficients (element_kernels.cuh)
//    precomputed at construction from the T-rounded vertices — 12 scalars
//    instead of the reference's 12 coordinates + 2 Lame values;
//  * Dirichlet mask bits ride in bits 28..30 of the connectivity word, so the
//    gather/scatter need no extra loads (masked inputs read as 0, masked
//    outputs skipped: ebe_operator.hpp:154-155,182);
//  * f starts as the masked identity (ebe_operator.hpp:96-110) and element
//    contributions land through fire-and-forget vector REDs in L2.
#include <algorithm>
#include <climits>
#include <parallel/algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <tuple>
#include <type_traits>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {

namespace {

template <typename T> struct Vec4Of;
template <typename T> using float2_or = typename std::conditional<sizeof(T) == 4, float2, T>::type;
template <> struct Vec4Of<float> { using type = float4; };
template <> struct Vec4Of<double> { using type = double2; };

// ---- cp.async helpers (Ampere+ LDGSTS; zero-fill when src_size == 0) --------
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int src_size, int bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_size) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src_size) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Persistent, software-pipelined element sweep (generic: any batch width, multi-pass beyond 32 cases).
// Each lane group (TPE threads, CPT cases each) walks elements e, e+G, e+2G..
// (G = all groups of the grid, so the grid sweeps a contiguous, L2-resident
// window of the Morton-ordered mesh). While element e is computed from shared
// memory, the gathers of element e+G are already in flight as cp.async into
// the other stage (double buffering): the L2 gather latency hides behind the
// ~500-flop element product instead of stalling it. Constrained dofs are
// zero-filled by the copy engine (src-size 0) — no branches, no extra loads.
template <typename T, typename V, int NPE, int CS>
__global__ void __launch_bounds__(128, 3)
k_ebe_pipe(const int32_t* __restrict__ conn, const T* __restrict__ coef, int32_t e_begin, int32_t n_elems,
           int tpe_shift, int32_t batch, int32_t col_base, const T* __restrict__ u, T* __restrict__ f) {
  using O = LaneOps<V>;
  constexpr int CPT = O::kCols;
  constexpr int NIN = NPE * 3;
  constexpr int NT = 128;
  constexpr int TPC = 16 / sizeof(T);  // scalars per 16-byte chunk
  constexpr int CHUNKS = 12 / TPC;     // coefficient record = 3 (fp32) / 6 (fp64) chunks
  extern __shared__ __align__(16) unsigned char smem[];
  const int TPE = 1 << tpe_shift;
  const int groups = NT >> tpe_shift;
  V* ubuf = reinterpret_cast<V*>(smem);                                   // [2][NIN][NT]
  T* cbuf = reinterpret_cast<T*>(smem + 2 * NIN * NT * sizeof(V));         // [2][groups][12]
  int32_t* nbuf = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(cbuf) +
                                             2 * groups * 12 * sizeof(T));  // [2][groups][CS]
  const int grp = threadIdx.x >> tpe_shift;
  const int lane = threadIdx.x & (TPE - 1);
  const int G = gridDim.x * groups;
  const int col = col_base + lane * CPT;
  const bool colok = col < batch;
  int e = e_begin + blockIdx.x * groups + grp;

  auto issue = [&](int ee, int stage) {
    if (ee < n_elems) {
      int32_t nd[CS];
      const int4* c4 = reinterpret_cast<const int4*>(conn + static_cast<size_t>(ee) * CS);
#pragma unroll
      for (int q = 0; q < CS / 4; ++q) {
        const int4 v = __ldg(c4 + q);
        nd[4 * q] = v.x; nd[4 * q + 1] = v.y; nd[4 * q + 2] = v.z; nd[4 * q + 3] = v.w;
        if (lane == 0) reinterpret_cast<int4*>(nbuf + (stage * groups + grp) * CS)[q] = v;
      }
      for (int q = lane; q < CHUNKS; q += TPE)
        cp_async(cbuf + (stage * groups + grp) * 12 + q * TPC, coef + static_cast<size_t>(ee) * 12 + q * TPC, 16, 16);
#pragma unroll
      for (int a = 0; a < NPE; ++a) {
        const uint32_t node = static_cast<uint32_t>(nd[a]) & 0x0FFFFFFFu;
        const T* row = u + static_cast<size_t>(3 * node) * batch + col;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const bool live = colok && !((nd[a] >> (28 + c)) & 1);
          cp_async(ubuf + (stage * NIN + a * 3 + c) * NT + threadIdx.x, live ? row + c * batch : u,
                   live ? int(sizeof(V)) : 0, sizeof(V));
        }
      }
    }
    cp_async_commit();
  };

  issue(e, 0);
  int s = 0;
  while (__any_sync(0xffffffffu, e < n_elems)) {
    const int en = e + G;
    issue(en, s ^ 1);
    cp_async_wait<1>();
    __syncwarp();
    if (e < n_elems && colok) {
      const T* cf = cbuf + (s * groups + grp) * 12;
      V b[3][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) b[k][d] = O::splat(cf[3 * k + d]);
      const V lp = O::splat(cf[9]), mp = O::splat(cf[10]);
      V uu[NPE][3];
#pragma unroll
      for (int q = 0; q < NIN; ++q) uu[q / 3][q % 3] = ubuf[(s * NIN + q) * NT + threadIdx.x];
      V ff[NPE][3];
      if constexpr (NPE == 10) tet10_product<V>(uu, b, lp, mp, ff);
      else tet4_product<V>(uu, b, lp, mp, ff);
      const int32_t* nd = nbuf + (s * groups + grp) * CS;
#pragma unroll
      for (int a = 0; a < NPE; ++a) {
        const int32_t w = nd[a];
        T* row = f + static_cast<size_t>(3 * (static_cast<uint32_t>(w) & 0x0FFFFFFFu)) * batch + col;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (!((w >> (28 + c)) & 1)) red_lane(reinterpret_cast<V*>(row + c * batch), ff[a][c]);
      }
    }
    __syncwarp();
    e = en;
    s ^= 1;
  }
  cp_async_wait<0>();
}

template <typename V> struct __align__(2 * sizeof(V)) V2Of { V a, b; };

// predicated fire-and-forget accumulation (no branch): skip when `off` != 0
__device__ __forceinline__ void red_pred(float2* p, float2 v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %3, 0; @q red.global.add.v2.f32 [%0], {%1, %2}; }" ::"l"(p),
               "f"(v.x), "f"(v.y), "r"(skip)
               : "memory");
}
__device__ __forceinline__ void red_pred(float* p, float v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %2, 0; @q red.global.add.f32 [%0], %1; }" ::"l"(p), "f"(v),
               "r"(skip)
               : "memory");
}
__device__ __forceinline__ void red_pred(double* p, double v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %2, 0; @q red.global.add.f64 [%0], %1; }" ::"l"(p), "d"(v),
               "r"(skip)
               : "memory");
}

// Production sweep: k_ebe_pipe specialised on the batch width B (<= 32), so
// every per-dof offset (c * B, lane column) is an immediate and one address is
// formed per node. Connectivity words hold 3 * node; word NPE holds the
// element's dof-mask bits (bit 3a+c). The next element's connectivity is
// prefetched one iteration ahead in registers, so the cp.async gathers issue
// without waiting on L2.
template <typename T, typename V, int NPE, int CS, int B>
__global__ void __launch_bounds__(128, 3)
k_ebe_fast(const int32_t* __restrict__ conn, const T* __restrict__ coef, int32_t e_begin, int32_t n_elems,
           const T* __restrict__ u, T* __restrict__ f) {
  using O = LaneOps<V>;
  constexpr int CPT = O::kCols;
  constexpr int NIN = NPE * 3;
  constexpr int NT = 128;
  constexpr int TPE = (B + CPT - 1) / CPT <= 1 ? 1 : ((B + CPT - 1) / CPT <= 2 ? 2 : ((B + CPT - 1) / CPT <= 4 ? 4 : ((B + CPT - 1) / CPT <= 8 ? 8 : 16)));
  constexpr int GROUPS = NT / TPE;
  constexpr int TPC = 16 / sizeof(T);
  constexpr int CHUNKS = 12 / TPC;
  extern __shared__ __align__(16) unsigned char smem[];
  V* ubuf = reinterpret_cast<V*>(smem);                                  // [2][NIN][NT]
  T* cbuf = reinterpret_cast<T*>(smem + 2 * NIN * NT * sizeof(V));        // [2][GROUPS][12]
  int32_t* nbuf = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(cbuf) +
                                             2 * GROUPS * 12 * sizeof(T));  // [2][GROUPS][CS]
  const int grp = threadIdx.x / TPE;
  const int lane = threadIdx.x % TPE;
  const int G = gridDim.x * GROUPS;
  const int col = lane * CPT;
  const bool colok = col < B;
  constexpr bool kFull = TPE * CPT == B;  // every lane's columns exist
  int e = e_begin + blockIdx.x * GROUPS + grp;

  int32_t nd[CS];  // connectivity of the element whose gathers issue next
  auto load_conn = [&](int ee) {
    if (ee < n_elems) {
      const int4* c4 = reinterpret_cast<const int4*>(conn + static_cast<size_t>(ee) * CS);
#pragma unroll
      for (int q = 0; q < CS / 4; ++q) {
        const int4 v = __ldg(c4 + q);
        nd[4 * q] = v.x; nd[4 * q + 1] = v.y; nd[4 * q + 2] = v.z; nd[4 * q + 3] = v.w;
      }
    }
  };
  auto issue = [&](int ee, int stage) {
    if (ee < n_elems) {
      if (lane == 0) {
        int4* dst = reinterpret_cast<int4*>(nbuf + (stage * GROUPS + grp) * CS);
#pragma unroll
        for (int q = 0; q < CS / 4; ++q) dst[q] = make_int4(nd[4 * q], nd[4 * q + 1], nd[4 * q + 2], nd[4 * q + 3]);
      }
      for (int q = lane; q < CHUNKS; q += TPE)
        cp_async(cbuf + (stage * GROUPS + grp) * 12 + q * TPC, coef + static_cast<size_t>(ee) * 12 + q * TPC, 16, 16);
      V* dst = ubuf + stage * NIN * NT + 2 * threadIdx.x;  // dof q at [q/2][tid][q%2]
      const unsigned mw = static_cast<unsigned>(nd[NPE]);
      if (kFull && mw == 0u) {  // interior element, all columns live: no per-dof predicates
#pragma unroll
        for (int a = 0; a < NPE; ++a) {
          const T* row = u + static_cast<size_t>(static_cast<uint32_t>(nd[a])) * B + col;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            cp_async(dst + ((a * 3 + c) >> 1) * 2 * NT + ((a * 3 + c) & 1), row + c * B, int(sizeof(V)), sizeof(V));
        }
      } else {
        const unsigned live = colok ? ~mw : 0u;
#pragma unroll
        for (int a = 0; a < NPE; ++a) {
          const T* row = u + static_cast<size_t>(static_cast<uint32_t>(nd[a])) * B + col;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            cp_async(dst + ((a * 3 + c) >> 1) * 2 * NT + ((a * 3 + c) & 1), row + c * B,
                     ((live >> (3 * a + c)) & 1u) * int(sizeof(V)), sizeof(V));
        }
      }
    }
    cp_async_commit();
  };

  load_conn(e);
  issue(e, 0);
  load_conn(e + G);
  int s = 0;
  while (__any_sync(0xffffffffu, e < n_elems)) {
    const int en = e + G;
    issue(en, s ^ 1);
    load_conn(en + G);  // consumed by the next iteration's issue
    cp_async_wait<1>();
    __syncwarp();
    if (e < n_elems && colok) {
      const T* cf = cbuf + (s * GROUPS + grp) * 12;
      V b[3][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) b[k][d] = O::splat(cf[3 * k + d]);
      const V lp = O::splat(cf[9]), mp = O::splat(cf[10]);
      V uu[NPE][3];
      const V* src = ubuf + s * NIN * NT + 2 * threadIdx.x;
#pragma unroll
      for (int q = 0; q < NIN; q += 2) {
        V2Of<V> pr = *reinterpret_cast<const V2Of<V>*>(src + (q >> 1) * 2 * NT);
        uu[q / 3][q % 3] = pr.a;
        uu[(q + 1) / 3][(q + 1) % 3] = pr.b;
      }
      V ff[NPE][3];
      if constexpr (NPE == 10) tet10_product<V>(uu, b, lp, mp, ff);
      else tet4_product<V>(uu, b, lp, mp, ff);
      const int32_t* ndc = nbuf + (s * GROUPS + grp) * CS;
      const unsigned mk = static_cast<unsigned>(ndc[NPE]);
      if (mk == 0u) {
#pragma unroll
        for (int a = 0; a < NPE; ++a) {
          T* row = f + static_cast<size_t>(static_cast<uint32_t>(ndc[a])) * B + col;
#pragma unroll
          for (int c = 0; c < 3; ++c) red_lane(reinterpret_cast<V*>(row + c * B), ff[a][c]);
        }
      } else {
#pragma unroll
        for (int a = 0; a < NPE; ++a) {
          T* row = f + static_cast<size_t>(static_cast<uint32_t>(ndc[a])) * B + col;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            red_pred(reinterpret_cast<V*>(row + c * B), ff[a][c], (mk >> (3 * a + c)) & 1u);
        }
      }
    }
    __syncwarp();
    e = en;
    s ^= 1;
  }
  cp_async_wait<0>();
}

// f = mask ? u : 0, vectorised over the contiguous [dof][case] array.
template <typename T>
__global__ void k_masked_identity(const uint8_t* __restrict__ mask, int64_t n_vec, int32_t batch,
                                  const T* __restrict__ u, T* __restrict__ f) {
  using V4 = typename Vec4Of<T>::type;
  constexpr int W = sizeof(V4) / sizeof(T);
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_vec) return;
  const int64_t d = (i * W) / batch;  // batch % W == 0 on this path
  V4 v;
  if (__ldg(mask + d)) v = __ldg(reinterpret_cast<const V4*>(u) + i);
  else std::memset(&v, 0, sizeof v);
  reinterpret_cast<V4*>(f)[i] = v;
}
// f[dof][*] = u[dof][*] for the listed constrained dofs (after a memset of f):
// the identity rows of ebe_operator.hpp:96-110 without reading the whole of u
template <typename T>
__global__ void k_identity_rows(const int32_t* __restrict__ dofs, int32_t n_dofs, int32_t batch,
                                const T* __restrict__ u, T* __restrict__ f) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(n_dofs) * batch) return;
  const int64_t k = i / batch;
  const int64_t at = int64_t(dofs[k]) * batch + (i - k * batch);
  f[at] = u[at];
}

template <typename T>
__global__ void k_masked_identity_scalar(const uint8_t* __restrict__ mask, int64_t n, int32_t batch,
                                         const T* __restrict__ u, T* __restrict__ f) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  f[i] = __ldg(mask + i / batch) ? __ldg(u + i) : T(0);
}

// ---- block Jacobi setup (extract_block_jacobi, ebe_operator.hpp:288-313) ----
// K_aa = sum_q (w detJ) [ (l+m) g g^T + m |g|^2 I ], g = grad N_a(q) from b_k;
// the 4-point rule (element_stiffness.hpp:39-51) with w detJ = V/4.
template <int NPE>
__global__ void k_bj_diag(const int32_t* __restrict__ conn, int cs, const double* __restrict__ c64,
                          int32_t n_elems, double* __restrict__ diag) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n_elems) return;
  const double* c = c64 + 12 * e;
  double b[4][3];
  for (int d = 0; d < 3; ++d) {
    b[1][d] = c[d]; b[2][d] = c[3 + d]; b[3][d] = c[6 + d];
    b[0][d] = -(b[1][d] + b[2][d] + b[3][d]);
  }
  const double lv = c[9], mv = c[10];
  auto add = [&](int a, const double (&g)[3], double w) {
    const int32_t node = conn[e * cs + a] & 0x0FFFFFFF;
    const double gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
    double* dst = diag + 9 * static_cast<size_t>(node);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        atomicAdd(dst + 3 * i + j, w * ((lv + mv) * g[i] * g[j] + (i == j ? mv * gg : 0.0)));
  };
  if (NPE == 4) {
    for (int a = 0; a < 4; ++a) {
      const double g[3] = {b[a][0], b[a][1], b[a][2]};
      add(a, g, 1.0);
    }
    return;
  }
  const double A = 0.58541019662496845, B = 0.13819660112501051;
  const int ends[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  for (int a = 0; a < 10; ++a) {
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < 4; ++q) {
      double L[4] = {B, B, B, B};
      L[q] = A;  // point q has L_q = A (ordering irrelevant: all 4 points summed)
      double g[3];
      if (a < 4) {
        for (int d = 0; d < 3; ++d) g[d] = (4.0 * L[a] - 1.0) * b[a][d];
      } else {
        const int p = ends[a - 4][0], r = ends[a - 4][1];
        for (int d = 0; d < 3; ++d) g[d] = 4.0 * (L[p] * b[r][d] + L[r] * b[p][d]);
      }
      const double gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) acc[3 * i + j] += (lv + mv) * g[i] * g[j] + (i == j ? mv * gg : 0.0);
    }
    const int32_t node = conn[e * cs + a] & 0x0FFFFFFF;
    double* dst = diag + 9 * static_cast<size_t>(node);
    for (int i = 0; i < 9; ++i) atomicAdd(dst + i, 0.25 * acc[i]);
  }
}

// invert_node_block (block_jacobi.hpp:45-66): masked axes -> identity, then invert.
template <typename T>
__global__ void k_bj_invert(const double* __restrict__ diag, const uint8_t* __restrict__ mask,
                            int32_t n, T* __restrict__ inv, int* __restrict__ bad) {
  const int32_t node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= n) return;
  double m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = diag[9 * static_cast<size_t>(node) + 3 * i + j];
  if (mask)
    for (int i = 0; i < 3; ++i)
      if (mask[3 * static_cast<size_t>(node) + i]) {
        for (int j = 0; j < 3; ++j) m[i][j] = m[j][i] = 0.0;
        m[i][i] = 1.0;
      }
  double scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) scale = fmax(scale, fabs(m[i][j]));
  const double d = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                   m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                   m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  if (scale == 0.0 || fabs(d) <= 1e-300 || d == 0.0) {
    atomicMin(bad, node);
    return;
  }
  const double id = 1.0 / d;
  double r[9];
  r[0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) * id;
  r[1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * id;
  r[2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * id;
  r[3] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) * id;
  r[4] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * id;
  r[5] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * id;
  r[6] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) * id;
  r[7] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * id;
  r[8] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * id;
  for (int q = 0; q < 9; ++q) inv[9 * static_cast<size_t>(node) + q] = static_cast<T>(r[q]);
}

int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

template <typename T, typename V, int NPE, int CS>
void launch_pipe(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int32_t e0 = 0,
                 int32_t e1 = -1) {
  if (e1 < 0) e1 = op.n_elems;
  if (e1 <= e0) return;
  constexpr int CPT = LaneOps<V>::kCols;
  constexpr int NT = 128;
  const int nct = (batch + CPT - 1) / CPT;
  const int tpe = std::min(pow2ceil(nct), 16);
  int shift = 0;
  while ((1 << shift) < tpe) ++shift;
  const int groups = NT / tpe;
  const size_t smem = 2 * size_t(NPE) * 3 * NT * sizeof(V) + 2 * size_t(groups) * 12 * sizeof(T) +
                      2 * size_t(groups) * CS * sizeof(int32_t);
  auto kern = k_ebe_pipe<T, V, NPE, CS>;
  static thread_local int cached_sms = 0;
  if (!cached_sms) {
    int dev = 0;
    TS_CUDA(cudaGetDevice(&dev));
    TS_CUDA(cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  per_sm = std::max(per_sm, 1);
  const int nct_passes = (nct + tpe - 1) / tpe;
  const int64_t need = (int64_t(e1 - e0) + groups - 1) / groups;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(cached_sms) * per_sm)));
  for (int p = 0; p < nct_passes; ++p) {
    kern<<<grid, NT, smem, s>>>(op.conn.get(), reinterpret_cast<const T*>(op.coef.get()), e0, e1,
                                 shift, batch, p * tpe * CPT, u, f);
    TS_CUDA_LAUNCH();
  }
}

template <typename T, typename V, int NPE, int CS, int B>
bool launch_fast_b(const ts_ebe& op, const T* u, T* f, cudaStream_t s, int32_t e0, int32_t e1) {
  constexpr int CPT = LaneOps<V>::kCols;
  constexpr int NT = 128;
  constexpr int nct = (B + CPT - 1) / CPT;
  if constexpr (nct > 16) {
    return false;  // wider than one 16-lane group: generic multi-pass kernel
  } else {
    constexpr int TPE = nct <= 1 ? 1 : nct <= 2 ? 2 : nct <= 4 ? 4 : nct <= 8 ? 8 : 16;
    constexpr int GROUPS = NT / TPE;
    const size_t smem = 2 * size_t(NPE) * 3 * NT * sizeof(V) + 2 * size_t(GROUPS) * 12 * sizeof(T) +
                        2 * size_t(GROUPS) * CS * sizeof(int32_t);
    auto kern = k_ebe_fast<T, V, NPE, CS, B>;
    const KernelFit fit = kernel_fit<k_ebe_fast<T, V, NPE, CS, B>>(NT, smem);
    const int sms = fit.sms, per_sm = std::max(fit.per_sm, 1);
    if (e1 <= e0) return true;
    const int64_t need = (int64_t(e1 - e0) + GROUPS - 1) / GROUPS;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * per_sm)));
    kern<<<grid, NT, smem, s>>>(op.conn3.get(), reinterpret_cast<const T*>(op.coef.get()), e0, e1, u, f);
    TS_CUDA_LAUNCH();
    return true;
  }
}

template <typename T, typename V, int NPE, int CS>
bool launch_fast(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int32_t e0, int32_t e1) {
  switch (batch) {
    case 1: return launch_fast_b<T, V, NPE, CS, 1>(op, u, f, s, e0, e1);
    case 2: return launch_fast_b<T, V, NPE, CS, 2>(op, u, f, s, e0, e1);
    case 4: return launch_fast_b<T, V, NPE, CS, 4>(op, u, f, s, e0, e1);
    case 8: return launch_fast_b<T, V, NPE, CS, 8>(op, u, f, s, e0, e1);
    case 16: return launch_fast_b<T, V, NPE, CS, 16>(op, u, f, s, e0, e1);
    case 20: return launch_fast_b<T, V, NPE, CS, 20>(op, u, f, s, e0, e1);
    case 32: return launch_fast_b<T, V, NPE, CS, 32>(op, u, f, s, e0, e1);
    default: return false;
  }
}

// part: -1 = every element, 0 = boundary group [0, group_split), 1 = interior
// group [group_split, E) (partitioned operators, dist_solver.cu); init: write
// the masked identity into f first.
template <typename T>
void apply_t(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int part, bool init) {
  const int64_t n = 3 * static_cast<int64_t>(op.n_nodes) * batch;
  // identity rows for constrained dofs, zero elsewhere (ebe_operator.hpp:96-110)
  if (init) {
    if (!op.has_mask || op.n_masked_dofs * 10 < 3 * int64_t(op.n_nodes)) {
      // write-only zero fill, then the (few) constrained rows copied from u
      TS_CUDA(cudaMemsetAsync(f, 0, n * sizeof(T), s));
      if (op.has_mask && op.n_masked_dofs > 0) {
        k_identity_rows<T><<<grid_for(int64_t(op.n_masked_dofs) * batch, 256), 256, 0, s>>>(
            op.masked_dofs.get(), op.n_masked_dofs, batch, u, f);
        TS_CUDA_LAUNCH();
      }
    } else {
      constexpr int W = sizeof(typename Vec4Of<T>::type) / sizeof(T);
      if (batch % W == 0)
        k_masked_identity<T><<<grid_for(n / W, 256), 256, 0, s>>>(op.mask.get(), n / W, batch, u, f);
      else
        k_masked_identity_scalar<T><<<grid_for(n, 256), 256, 0, s>>>(op.mask.get(), n, batch, u, f);
      TS_CUDA_LAUNCH();
    }
  }
  if (op.timing) TS_CUDA(cudaEventRecord(op.ev0, s));  // times the element sweep only
  const int32_t e0 = part == 1 ? op.group_split : 0, e1 = part == 0 ? op.group_split : op.n_elems;
  if (e1 <= e0) {
    if (op.timing) TS_CUDA(cudaEventRecord(op.ev1, s));
    return;
  }
  bool done = false;
  if (op.deterministic) {  // order-fixed colored sweep (reference bitwise contract, test_ebe.cpp:254-317)
    ebe_color_apply(op, u, f, batch, s, part);
    done = true;
  }
  // Default dispatch (6, measured: profiles/r01_ebe_tile.txt, r01_ebe_pair_ncu.txt): the face-pair sweep
  // (ebe_pair.cu) for every batch width it covers (1, 2, 4, 8, 16), else the element-parallel sweep.
  if (!done && op.fan) done = ebe_fan_apply(op, u, f, batch, s, part);
  if (!done && op.pair) done = ebe_pair_apply(op, u, f, batch, s, part);
  if (!done && op.kernel >= 3)
    done = (op.order == 2)
               ? (sizeof(T) == 4 && batch % 2 == 0 ? launch_fast<T, float2_or<T>, 10, 12>(op, u, f, batch, s, e0, e1)
                                                   : launch_fast<T, T, 10, 12>(op, u, f, batch, s, e0, e1))
               : (sizeof(T) == 4 && batch % 2 == 0 ? launch_fast<T, float2_or<T>, 4, 8>(op, u, f, batch, s, e0, e1)
                                                   : launch_fast<T, T, 4, 8>(op, u, f, batch, s, e0, e1));
  if (!done) {  // any batch width: the generic pipelined sweep over the element range
    if (op.order == 2) {
      if (sizeof(T) == 4 && batch % 2 == 0) launch_pipe<float, float2, 10, 12>(op, reinterpret_cast<const float*>(u), reinterpret_cast<float*>(f), batch, s, e0, e1);
      else launch_pipe<T, T, 10, 12>(op, u, f, batch, s, e0, e1);
    } else {
      if (sizeof(T) == 4 && batch % 2 == 0) launch_pipe<float, float2, 4, 4>(op, reinterpret_cast<const float*>(u), reinterpret_cast<float*>(f), batch, s, e0, e1);
      else launch_pipe<T, T, 4, 4>(op, u, f, batch, s, e0, e1);
    }
  }
  if (op.timing) TS_CUDA(cudaEventRecord(op.ev1, s));
}

void det_inv3(const double j[3][3], double inv[3][3], double* det) {
  const double d = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                   j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                   j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
  *det = d;
  if (d == 0.0) {
    std::memset(inv, 0, sizeof(double) * 9);
    return;
  }
  const double id = 1.0 / d;
  inv[0][0] = (j[1][1] * j[2][2] - j[1][2] * j[2][1]) * id;
  inv[0][1] = (j[0][2] * j[2][1] - j[0][1] * j[2][2]) * id;
  inv[0][2] = (j[0][1] * j[1][2] - j[0][2] * j[1][1]) * id;
  inv[1][0] = (j[1][2] * j[2][0] - j[1][0] * j[2][2]) * id;
  inv[1][1] = (j[0][0] * j[2][2] - j[0][2] * j[2][0]) * id;
  inv[1][2] = (j[0][2] * j[1][0] - j[0][0] * j[1][2]) * id;
  inv[2][0] = (j[1][0] * j[2][1] - j[1][1] * j[2][0]) * id;
  inv[2][1] = (j[0][1] * j[2][0] - j[0][0] * j[2][1]) * id;
  inv[2][2] = (j[0][0] * j[1][1] - j[0][1] * j[1][0]) * id;
}

}  // namespace

void ebe_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s) {
  NvtxRange nv("ebe apply");
  if (batch < 1) validation("ebe apply: batch must be >= 1");
  if (u == f) validation("ebe apply: input and output must not alias");
  if (op.prec == 32) apply_t<float>(op, static_cast<const float*>(u), static_cast<float*>(f), batch, s, -1, true);
  else apply_t<double>(op, static_cast<const double*>(u), static_cast<double*>(f), batch, s, -1, true);
}

int ebe_launches_per_apply(const ts_ebe& op, int32_t batch) {
  // masked-identity init: memset (copy engine) + identity-row kernel, or one masked-identity kernel
  const int init = op.has_mask && op.n_masked_dofs > 0 ? 1 : 0;
  if (op.deterministic) {
    int n = 0;
    for (size_t k = 0; k + 1 < op.color->color_ptr.size(); ++k) n += op.color->color_ptr[k + 1] > op.color->color_ptr[k];
    return init + n;
  }
  if (op.fan) {
    const int p = ebe_fan_launches(op, batch);
    if (p >= 0) return init + p;
  }
  if (op.pair) {
    const int p = ebe_pair_launches(op, batch);
    if (p >= 0) return init + p;
  }
  const int cpt = op.prec == 32 && batch % 2 == 0 ? 2 : 1;
  const int nct = (batch + cpt - 1) / cpt;
  const bool fast = op.kernel >= 3 && nct <= 16 &&
                    (batch == 1 || batch == 2 || batch == 4 || batch == 8 || batch == 16 || batch == 20 || batch == 32);
  const int groups = op.group_split > 0 && op.group_split < op.n_elems ? 2 : 1;
  if (fast) return init + groups;
  const int tpe = std::min(pow2ceil(nct), 16);
  return init + groups * ((nct + tpe - 1) / tpe);
}

void ebe_apply_part(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part, bool init) {
  if (batch < 1) validation("ebe apply: batch must be >= 1");
  if (u == f) validation("ebe apply: input and output must not alias");
  if (op.prec == 32) apply_t<float>(op, static_cast<const float*>(u), static_cast<float*>(f), batch, s, part, init);
  else apply_t<double>(op, static_cast<const double*>(u), static_cast<double*>(f), batch, s, part, init);
}

void ebe_diag_blocks(const ts_ebe& op, double* diag, cudaStream_t s) {
  if (op.coef64.size() != 12 * static_cast<size_t>(op.n_elems))
    validation("block jacobi: operator setup data released (level-set inner operators keep only device state)");
  DevBuf<double> c64;
  c64.upload(op.coef64, s);
  setup_mark("bj: upload records");
  TS_CUDA(cudaMemsetAsync(diag, 0, 9 * static_cast<size_t>(op.n_nodes) * sizeof(double), s));
  if (op.n_elems > 0) {
    if (op.order == 2)
      k_bj_diag<10><<<grid_for(op.n_elems, 128), 128, 0, s>>>(op.conn.get(), op.conn_stride, c64.get(), op.n_elems,
                                                              diag);
    else
      k_bj_diag<4><<<grid_for(op.n_elems, 128), 128, 0, s>>>(op.conn.get(), op.conn_stride, c64.get(), op.n_elems,
                                                             diag);
    TS_CUDA_LAUNCH();
  }
  TS_CUDA(cudaStreamSynchronize(s));  // c64 is released on return
}

void bj_invert(const double* diag, const uint8_t* mask, int32_t n, int prec, void* inv_dev, cudaStream_t s) {
  DevBuf<int32_t> bad(1);
  const int init = INT32_MAX;
  TS_CUDA(cudaMemcpyAsync(bad.get(), &init, sizeof(int), cudaMemcpyHostToDevice, s));
  if (prec == 32)
    k_bj_invert<float><<<grid_for(n, 128), 128, 0, s>>>(diag, mask, n, static_cast<float*>(inv_dev), bad.get());
  else
    k_bj_invert<double><<<grid_for(n, 128), 128, 0, s>>>(diag, mask, n, static_cast<double*>(inv_dev), bad.get());
  TS_CUDA_LAUNCH();
  int hb = 0;
  TS_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  TS_CUDA(cudaStreamSynchronize(s));
  if (hb != INT32_MAX) validation("block jacobi: singular diagonal block at node " + std::to_string(hb));
}

void ebe_block_jacobi(const ts_ebe& op, void* inv_dev, cudaStream_t s) {
  DevBuf<double> diag(9 * static_cast<size_t>(op.n_nodes));
  ebe_diag_blocks(op, diag.get(), s);
  bj_invert(diag.get(), op.has_mask ? op.mask.get() : nullptr, op.n_nodes, op.prec, inv_dev, s);
}

int ebe_slab_count() {
  static const int n = [] {
    const char* e = std::getenv("TSGPU_EBE_SLABS");
    const int v = e ? std::atoi(e) : kEbeSlabs;
    return std::max(1, std::min(255, v));
  }();
  return n;
}

ts_ebe* ebe_create(const Mesh& m, int order, int32_t n_mat, const double* lambda, const double* mu,
                   const uint8_t* dof_mask, int prec, const uint8_t* elem_group, int kernel_override,
                   std::vector<int32_t>* element_order, PairTopology* pair_topology) {
  if (order != 1 && order != 2) validation("ebe: order must be 1 or 2");
  if (prec != 32 && prec != 64) validation("ebe: precision must be 32 or 64");
  require_device();
  auto op = std::make_unique<ts_ebe>();
  op->order = order;
  op->prec = prec;
  op->npe = order == 1 ? 4 : 10;
  op->conn_stride = order == 1 ? 4 : 12;
  op->n_nodes = order == 1 ? m.vertex_count : m.n_nodes();
  op->n_elems = m.n_elems();
  op->n_vertices = m.vertex_count;
  op->n_slabs = ebe_slab_count();
  if (op->n_nodes >= (1 << 28)) validation("ebe: more than 2^28 nodes per device is not supported");
  op->has_mask = dof_mask != nullptr;
  const int npe = op->npe, cs = op->conn_stride;
  const size_t E = static_cast<size_t>(op->n_elems);
  if (dof_mask) op->host_mask.assign(dof_mask, dof_mask + 3 * static_cast<size_t>(op->n_nodes));
  auto rnd = [prec](double x) { return prec == 32 ? static_cast<double>(static_cast<float>(x)) : x; };
  // validation first (exceptions stay out of the parallel loops): find the first bad element in
  // parallel, then report it exactly as a sequential scan would
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
  for (int64_t e = 0; e < int64_t(E); ++e) {
    const int32_t mid = m.material_id[e];
    bool bad = mid < 0 || mid >= n_mat;
    for (int a = 0; a < npe; ++a) {
      const int32_t node = m.tets10[10 * e + a];
      bad |= node < 0 || node >= op->n_nodes;
    }
    if (bad) first_bad = std::min(first_bad, e);
  }
  if (first_bad != INT64_MAX) {
    const size_t e = static_cast<size_t>(first_bad);
    const int32_t mid = m.material_id[e];
    if (mid < 0 || mid >= n_mat)
      validation("ebe: element " + std::to_string(e) + " references material " + std::to_string(mid) +
                 " but only " + std::to_string(n_mat) + " defined");
    for (int a = 0; a < npe; ++a) {
      const int32_t node = m.tets10[10 * e + a];
      if (node < 0 || node >= op->n_nodes)
        validation("ebe: element " + std::to_string(e) + " references node " + std::to_string(node) +
                   " out of range");
    }
  }
  setup_mark("ebe: validate");
  // Element order: (group, slab, Morton key, id). A partitioned operator keeps
  // its boundary elements (group 0) ahead of the interior ones so the two sweep
  // separately; within a group, elements go in kSlabs slabs of their lowest
  // vertex id, then Morton (Z-order) of centroids. The slabs make node first /
  // last use monotone in node id for meshes numbered along an axis (the box
  // generator, most mesh tools), which lets the host-buffer apply stream u in
  // and f out while it sweeps (ebe_stream.cu); inside a slab the Morton order
  // keeps gathers and scatters L2-local.
  HostVec<int32_t> ord(E);
  {
    const bool reuse = element_order && element_order->size() == E;
    if (reuse) {  // the level set's other operators share one element order
      std::copy(element_order->begin(), element_order->end(), ord.begin());
    } else {
      HostVec<double> cen(3 * E);
#pragma omp parallel for schedule(static)
      for (size_t e = 0; e < E; ++e)
        for (int c = 0; c < 3; ++c) {
          double x = 0.0;
          for (int a = 0; a < 4; ++a) x += m.coords[3 * static_cast<size_t>(m.tets10[10 * e + a]) + c];
          cen[3 * e + c] = 0.25 * x;
        }
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (size_t e = 0; e < E; ++e)
        for (int c = 0; c < 3; ++c) {
          lo[c] = std::min(lo[c], cen[3 * e + c]);
          hi[c] = std::max(hi[c], cen[3 * e + c]);
        }
      auto spread = [](uint64_t v) {
        v &= 0x1FFFFF;
        v = (v | v << 32) & 0x1F00000000FFFFULL;
        v = (v | v << 16) & 0x1F0000FF0000FFULL;
        v = (v | v << 8) & 0x100F00F00F00F00FULL;
        v = (v | v << 4) & 0x10C30C30C30C30C3ULL;
        v = (v | v << 2) & 0x1249249249249249ULL;
        return v;
      };
      double ext = 0.0;
      for (int c = 0; c < 3; ++c) ext = std::max(ext, hi[c] - lo[c]);
      const double scale = ext > 0.0 ? double((1 << 20) - 1) / ext : 0.0;
      const int64_t vmax = std::max<int64_t>(1, m.vertex_count);
      HostVec<std::tuple<uint8_t, uint8_t, uint64_t, int32_t>> key(E);
#pragma omp parallel for schedule(static)
      for (size_t e = 0; e < E; ++e) {
        uint64_t k = 0;
        for (int c = 0; c < 3; ++c) k |= spread(static_cast<uint64_t>((cen[3 * e + c] - lo[c]) * scale)) << c;
        int32_t vlo = m.tets10[10 * e];
        for (int a = 1; a < 4; ++a) vlo = std::min(vlo, m.tets10[10 * e + a]);
        const auto slab = static_cast<uint8_t>(ebe_slab_of(vlo, vmax, op->n_slabs));
        key[e] = {elem_group ? elem_group[e] : uint8_t(0), slab, k, static_cast<int32_t>(e)};
      }
      __gnu_parallel::sort(key.begin(), key.end());
#pragma omp parallel for schedule(static)
      for (size_t i = 0; i < E; ++i) ord[i] = std::get<3>(key[i]);
      if (element_order) element_order->assign(ord.begin(), ord.end());
    }
    op->group_split = 0;
    if (elem_group) {
      for (size_t i = 0; i < E; ++i)
        if (elem_group[ord[i]] == 0) op->group_split = static_cast<int32_t>(i + 1);
    } else {
      op->group_split = static_cast<int32_t>(E);
    }
  }
  setup_mark("ebe: element order");
  // element records, written straight into sweep order (no zero fill: every
  // slot, padding included, is written by the parallel loop that first touches it)
  HostVec<int32_t> conn(E * cs);
  op->host_conn.resize(E * npe);
  op->coef64.resize(E * 12);
  op->elem_order.assign(ord.begin(), ord.end());
  const size_t ts = prec == 32 ? 4 : 8;
  HostVec<unsigned char> coef(E * 12 * ts);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < E; ++i) {
    const size_t e = static_cast<size_t>(ord[i]);
    const int32_t mid = m.material_id[e];
    const int32_t* t = m.tets10.data() + 10 * e;
    for (int a = 0; a < npe; ++a) {
      const int32_t node = t[a];
      int32_t word = node;
      if (dof_mask)
        for (int c = 0; c < 3; ++c)
          if (dof_mask[3 * static_cast<size_t>(node) + c]) word |= 1 << (28 + c);
      conn[i * cs + a] = word;
      op->host_conn[i * npe + a] = node;
    }
    for (int a = npe; a < cs; ++a) conn[i * cs + a] = 0;
    // T-rounded vertices and Lame values (ebe_operator.hpp:54-62), geometry in fp64
    double v[4][3];
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 3; ++c) v[a][c] = rnd(m.coords[3 * static_cast<size_t>(t[a]) + c]);
    const double lam = rnd(lambda[mid]), mue = rnd(mu[mid]);
    double j[3][3], inv[3][3], det;
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) j[r][c] = v[c + 1][r] - v[0][r];
    det_inv3(j, inv, &det);
    const double vol = det / 6.0;
    double* c64 = op->coef64.data() + 12 * i;
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) c64[3 * k + d] = inv[k][d];  // b_{k+1} = row k of J^-1
    c64[9] = lam * vol;
    c64[10] = mue * vol;
    c64[11] = vol;
    const double scale = order == 2 ? 1.0 / 20.0 : 1.0;
    double rec[12];
    for (int q = 0; q < 9; ++q) rec[q] = c64[q];
    rec[9] = lam * vol * scale;
    rec[10] = mue * vol * scale;
    rec[11] = 0.0;
    for (int q = 0; q < 12; ++q) {
      if (prec == 32) {
        const float x = static_cast<float>(rec[q]);
        std::memcpy(coef.data() + (12 * i + q) * ts, &x, 4);
      } else {
        std::memcpy(coef.data() + (12 * i + q) * ts, &rec[q], 8);
      }
    }
  }
  setup_mark("ebe: element records");
  if (kernel_override >= 0) op->kernel = kernel_override;
  else if (const char* k = std::getenv("TSGPU_EBE_KERNEL"))
    op->kernel = std::string(k) == "pipe" ? 2 : std::string(k) == "fast" ? 3 : std::string(k) == "pair" ? 7
               : std::string(k) == "fan" ? 8 : 6;
  const char* kenv = std::getenv("TSGPU_EBE_KERNEL");
  const bool colored = kernel_override < 0 && kenv && std::string(kenv) == "color";
  {
    // fast-kernel layout: 3*node per local node, then the dof-mask word (bit 3a+c)
    const int cs3 = order == 1 ? 8 : 12;
    HostVec<int32_t> conn3(E * cs3);
#pragma omp parallel for schedule(static)
    for (size_t e = 0; e < E; ++e) {
      for (int a = npe + 1; a < cs3; ++a) conn3[e * cs3 + a] = 0;
      uint32_t mw = 0;
      for (int a = 0; a < npe; ++a) {
        const int32_t w = conn[e * cs + a];
        conn3[e * cs3 + a] = 3 * (w & 0x0FFFFFFF);
        for (int c = 0; c < 3; ++c)
          if ((w >> (28 + c)) & 1) mw |= 1u << (3 * a + c);
      }
      conn3[e * cs3 + npe] = static_cast<int32_t>(mw);
    }
    op->conn3.upload(conn3);
  }
  setup_mark("ebe: conn3");
  // face pairs by default; edge fans (tet10) on request (TSGPU_EBE_KERNEL=fan; measured in
  // faster at r = 1, slower at r >= 4 on the FP-latency-bound sweep)
  const bool fans = order == 2 && op->kernel == 8;
  if (fans) build_fan_plan(*op, m, conn, cs, op->coef64, prec == 32);
  setup_mark("ebe: fan plan");
  if (!fans && (op->kernel == 7 || op->kernel == 6 || op->kernel == 8))  // (tet4 under "fan": pairs)
    build_pair_plan(*op, m, conn, cs, op->coef64, prec == 32, pair_topology);
  setup_mark("ebe: pair plan");
  op->conn.upload(conn);
  op->coef.upload(coef);
  if (dof_mask) {
    op->mask.upload(op->host_mask);
    std::vector<int32_t> md;
    for (size_t d = 0; d < op->host_mask.size(); ++d)
      if (op->host_mask[d]) md.push_back(static_cast<int32_t>(d));
    op->n_masked_dofs = static_cast<int32_t>(md.size());
    op->masked_dofs.upload(md);
  }
  TS_CUDA(cudaDeviceSynchronize());
  if (colored) ebe_set_deterministic(*op, true);
  return op.release();
}

}  // namespace tsg

ts_ebe::~ts_ebe() {
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
}
