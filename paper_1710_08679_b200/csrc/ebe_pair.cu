// ebe_pair.cu — EBE sweep over face-sharing element pairs (tet10).
//
// Same product as k_ebe_fast (ebe_operator.hpp:143-188 semantics, lean exact
// element math of element_kernels.cuh) but the unit of work is a PAIR of
// tetrahedra that share a face. The setup renumbers both elements' local nodes
// (a relabelling leaves K_e unchanged up to the same permutation of rows and
// columns; gradients are taken in the new order, the volume keeps the original
// orientation) so that the shared face is A's vertices (1,2,3) and B's vertices
// (0,1,2): the 6 shared nodes (3 vertices + 3 edge midpoints) then occupy fixed
// register slots. A lane group gathers 14 node rows instead of 20, computes A,
// reduces A's 4 unshared rows, keeps A's 6 face rows in registers, computes B,
// adds them and reduces B's 10 rows: 14 vector-RED node rows per pair instead
// of 20 — the L2 atomic traffic that bounds the element-parallel sweep drops by
// 30 % (profiles/r01_ebe_memory_paths.txt). Unpaired elements run as singles.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <vector>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {
namespace {

constexpr int kHasB = 1 << 31;

template <typename V>
struct __align__(2 * sizeof(V)) V2P {
  V a, b;
};

// an element's 12-scalar coefficient record from shared memory in 16-byte loads
__device__ __forceinline__ void load_rec(const float* p, float (&c)[12]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float4 v = reinterpret_cast<const float4*>(p)[i];
    c[4 * i] = v.x; c[4 * i + 1] = v.y; c[4 * i + 2] = v.z; c[4 * i + 3] = v.w;
  }
}
__device__ __forceinline__ void load_rec(const double* p, double (&c)[12]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double2 v = reinterpret_cast<const double2*>(p)[i];
    c[2 * i] = v.x; c[2 * i + 1] = v.y;
  }
}

// Slot geometry of a pair, per element order. A's shared face is its vertices
// (1,2,3) (+ edges 5, 9, 8 for tet10); B's is (0,1,2) (+ edges 4, 5, 6).
template <int NPE> struct PairGeo;
template <> struct PairGeo<10> {
  static constexpr int NR = 14;        // gathered node rows: A's 10, B's own 3,7,8,9
  static constexpr int WORDS = 16;     // NR node words, A mask bits, B own mask bits | hasB
  static constexpr int NA_OWN = 4, NFACE = 6, NB_OWN = 4;
  __host__ __device__ static constexpr int a_own(int k) { return k == 0 ? 0 : k == 1 ? 4 : k == 2 ? 6 : 7; }
  __host__ __device__ static constexpr int a_face(int k) { return k < 3 ? k + 1 : k == 3 ? 5 : k == 4 ? 9 : 8; }
  __host__ __device__ static constexpr int b_face(int k) { return k < 3 ? k : k + 1; }
  __host__ __device__ static constexpr int b_own(int k) { return k == 0 ? 3 : k + 6; }
  // gathered-row index of B's slot s
  __host__ __device__ static constexpr int b_row(int s) {
    return s == 0 ? 1 : s == 1 ? 2 : s == 2 ? 3 : s == 3 ? 10 : s == 4 ? 5 : s == 5 ? 9 : s == 6 ? 8 : s == 7 ? 11 : s == 8 ? 12 : 13;
  }
};
template <> struct PairGeo<4> {
  static constexpr int NR = 5;
  static constexpr int WORDS = 8;
  static constexpr int NA_OWN = 1, NFACE = 3, NB_OWN = 1;
  __host__ __device__ static constexpr int a_own(int) { return 0; }
  __host__ __device__ static constexpr int a_face(int k) { return k + 1; }
  __host__ __device__ static constexpr int b_face(int k) { return k; }
  __host__ __device__ static constexpr int b_own(int) { return 3; }
  __host__ __device__ static constexpr int b_row(int s) { return s < 3 ? s + 1 : 4; }
};

__device__ __forceinline__ void cpa(void* s, const void* g, int src, int bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
}

__device__ __forceinline__ void red_p(float2* p, float2 v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %3, 0; @q red.global.add.v2.f32 [%0], {%1, %2}; }" ::"l"(p),
               "f"(v.x), "f"(v.y), "r"(skip)
               : "memory");
}
__device__ __forceinline__ void red_p(float* p, float v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %2, 0; @q red.global.add.f32 [%0], %1; }" ::"l"(p), "f"(v), "r"(skip)
               : "memory");
}
__device__ __forceinline__ void red_p(double* p, double v, unsigned skip) {
  asm volatile("{ .reg .pred q; setp.eq.u32 q, %2, 0; @q red.global.add.f64 [%0], %1; }" ::"l"(p), "d"(v), "r"(skip)
               : "memory");
}

// Decomposition experiments (scripts/exp_pair_parts.sh; never in the product build):
// EXP_NORED keeps the products live but drops the scatter, EXP_NOGATHER drops the
// interior gathers (stale shared data), EXP_NOMATH replaces the element products by copies.
#if defined(EXP_NORED)
#define EXP_RED(p, v) (sink = O::add(sink, (v)))
#else
#define EXP_RED(p, v) red_lane(p, v)
#endif

__device__ __forceinline__ float lane_col(float2 v, int c) { return c ? v.y : v.x; }
__device__ __forceinline__ float lane_col(float v, int) { return v; }
__device__ __forceinline__ double lane_col(double v, int) { return v; }

// DOTS (the inner PCG's gamma, fused): every element adds p_e . (K_e p_e) over its unconstrained
// dofs — summed over elements that is (p, K p) restricted to the unconstrained dofs — per column
// in fp64 per lane; the block folds its lane groups in order into dpart[block][3][B] ((p,Ap) in
// slot 0; slots 1-2 zero: the constrained dofs' p.p and the norms come from elsewhere).
template <typename T, typename V, int NPE, int B, bool DOTS = false>
__global__ void __launch_bounds__(128, 2)
k_ebe_pair(const int32_t* __restrict__ pconn, const T* __restrict__ pcoef, int32_t p_begin, int32_t p_end,
           const T* __restrict__ u, T* __restrict__ f, int32_t* __restrict__ sched, double* __restrict__ dpart) {
  using O = LaneOps<V>;
  using Geo = PairGeo<NPE>;
  constexpr int CPT = O::kCols;
  [[maybe_unused]] V sink = O::zero();
  constexpr int NR = Geo::NR, NIN = (NR * 3 + 1) & ~1;  // gathered node rows / dofs per pair (even: pair slots)
  constexpr int kPairWords = Geo::WORDS;
  constexpr int MW = NR;                     // index of A's mask word (B's own follows)
  constexpr int NT = 128;
  constexpr int TPE = (B + CPT - 1) / CPT;
  static_assert(NT % TPE == 0, "lane groups must tile the block");
  constexpr int GROUPS = NT / TPE;
  constexpr int TPC = 16 / sizeof(T);
  constexpr int CHUNKS = 24 / TPC;  // two 12-scalar coefficient records
  extern __shared__ __align__(16) unsigned char smem[];
  V* ubuf = reinterpret_cast<V*>(smem);  // [2][NIN/2][NT][2]: dofs 2k, 2k+1 of a thread side by side
  T* cbuf = reinterpret_cast<T*>(smem + 2 * NIN * NT * sizeof(V));          // [2][GROUPS][24]
  int32_t* nbuf = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(cbuf) +
                                             2 * GROUPS * 24 * sizeof(T));  // [2][GROUPS][16]
  const int grp = threadIdx.x / TPE;
  const int lane = threadIdx.x % TPE;
  const int G = gridDim.x * GROUPS;
  // a thread's dof q lives at pair q/2, element q%2: one 2*sizeof(V) shared load serves two dofs
  auto slot = [](int q) { return (q >> 1) * 2 * NT + (q & 1); };
  auto dof = [](const V* base, int q) {
    const V2P<V> pr = *reinterpret_cast<const V2P<V>*>(base + (q >> 1) * 2 * NT);
    return (q & 1) ? pr.b : pr.a;
  };
  const int col = lane * CPT;
  int stat = p_begin + blockIdx.x * GROUPS + grp;  // static order: this group's next unit
  int e = 0;

  int32_t nd[kPairWords];
  double dacc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) dacc[c] = 0.0;
  // p_e . ff over the element's unconstrained dofs (p_e as gathered; mask bits per dof)
  auto edot = [&](const V (&uu)[NPE][3], const V (&ffe)[NPE][3], auto row_of, unsigned ma_, unsigned mb_,
                    bool interior) {
    V e = O::zero();
    if (interior) {
#pragma unroll
      for (int a = 0; a < NPE; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) e = O::fma(uu[a][c], ffe[a][c], e);
    } else {
#pragma unroll
      for (int a = 0; a < NPE; ++a) {
        const int r = row_of(a);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const unsigned m = r < NPE ? (ma_ >> (3 * r + c)) & 1u : (mb_ >> (3 * (r - NPE) + c)) & 1u;
          if (!m) e = O::fma(uu[a][c], ffe[a][c], e);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) dacc[c] += double(lane_col(e, c));
  };
  auto load_conn = [&](int ee) {
    if (ee < p_end) {
      const int4* c4 = reinterpret_cast<const int4*>(pconn + static_cast<size_t>(ee) * kPairWords);
#pragma unroll
      for (int q = 0; q < kPairWords / 4; ++q) {
        const int4 v = __ldg(c4 + q);
        nd[4 * q] = v.x; nd[4 * q + 1] = v.y; nd[4 * q + 2] = v.z; nd[4 * q + 3] = v.w;
      }
    }
  };
  auto issue = [&](int ee, int stage) {
    if (ee < p_end) {
      if (lane == 0) {
        int4* dst = reinterpret_cast<int4*>(nbuf + (stage * GROUPS + grp) * kPairWords);
#pragma unroll
        for (int q = 0; q < kPairWords / 4; ++q)
          dst[q] = make_int4(nd[4 * q], nd[4 * q + 1], nd[4 * q + 2], nd[4 * q + 3]);
      }
      for (int q = lane; q < CHUNKS; q += TPE)
        cpa(cbuf + (stage * GROUPS + grp) * 24 + q * TPC, pcoef + static_cast<size_t>(ee) * 24 + q * TPC, 16, 16);
      V* dst = ubuf + stage * NIN * NT + 2 * threadIdx.x;
      const unsigned ma = static_cast<unsigned>(nd[MW]), mb = static_cast<unsigned>(nd[MW + 1]);
      if (mb == unsigned(kHasB) && ma == 0u) {  // interior pair: no constrained dof, no per-dof predicates
#pragma unroll
        for (int a = 0; a < NR; ++a) {
          const T* row = u + static_cast<size_t>(static_cast<uint32_t>(nd[a])) * B + col;
#pragma unroll
#if !defined(EXP_NOGATHER)
          for (int c = 0; c < 3; ++c) cpa(dst + slot(a * 3 + c), row + c * B, int(sizeof(V)), sizeof(V));
#else
          (void)row;
#endif
        }
      } else {
#pragma unroll
        for (int a = 0; a < NR; ++a) {
          const T* row = u + static_cast<size_t>(static_cast<uint32_t>(nd[a])) * B + col;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const unsigned m = a < NPE ? (ma >> (3 * a + c)) & 1u : (mb >> (3 * (a - NPE) + c)) & 1u;
            cpa(dst + slot(a * 3 + c), row + c * B, m ? 0 : int(sizeof(V)), sizeof(V));
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // unit order: static strides (sched == nullptr) or warp chunks taken from a counter in sweep
  // order (sched), which keeps the front of concurrently swept units tight (no drift between lane
  // groups, so the rows they share stay in L2); a chunk's successor is claimed one chunk ahead
  constexpr int GPW = 32 / TPE < 1 ? 1 : 32 / TPE;  // lane groups per warp
#ifndef PAIR_J
#define PAIR_J 4
#endif
  constexpr int J = PAIR_J;                          // units per group per chunk
  const int gi = (threadIdx.x & 31) / TPE;
  int cbase = 0, k = 0, claim = 0;
  auto take = [&]() {  // lane 0 claims a chunk; the value is read (shfl) one chunk later
    if ((threadIdx.x & 31) == 0) claim = atomicAdd(sched, GPW * J);
  };
  auto next_unit = [&]() -> int {
    if (!sched) {
      const int r = stat;
      stat += G;
      return r;
    }
    const int r = p_begin + cbase + gi + k * GPW;
    if (++k == J) {
      k = 0;
      cbase = __shfl_sync(0xffffffffu, claim, 0);
      take();
    }
    return r;
  };
  if (sched) {
    take();
    cbase = __shfl_sync(0xffffffffu, claim, 0);
    take();
  }
  int e_cur = next_unit(), e_nxt = next_unit(), e_far = next_unit();
  load_conn(e_cur);
  issue(e_cur, 0);
  load_conn(e_nxt);
  e = e_cur;
  int s = 0;
  while (__any_sync(0xffffffffu, e < p_end)) {
    const int en = e_nxt;
    issue(en, s ^ 1);
    load_conn(e_far);
    e_nxt = e_far;
    e_far = next_unit();
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    if (e < p_end) {
      const T* cf = cbuf + (s * GROUPS + grp) * 24;
      const int32_t* w = nbuf + (s * GROUPS + grp) * kPairWords;
      const V* src = ubuf + s * NIN * NT + 2 * threadIdx.x;
      const unsigned ma = static_cast<unsigned>(w[MW]), mb = static_cast<unsigned>(w[MW + 1]);
      V carry[Geo::NFACE][3];  // A's face rows (= B's face rows)
      {
        T rec[12];
        load_rec(cf, rec);
        V b[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) b[k][d] = O::splat(rec[3 * k + d]);
        const V lp = O::splat(rec[9]), mp = O::splat(rec[10]);
        V uu[NPE][3];
#pragma unroll
        for (int a = 0; a < NPE; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) uu[a][c] = dof(src, a * 3 + c);
        V ff[NPE][3];
#if defined(EXP_NOMATH)
        for (int a = 0; a < NPE; ++a) for (int c = 0; c < 3; ++c) ff[a][c] = O::mul(uu[a][c], b[c][c]);
#else
        if constexpr (NPE == 10) tet10_product<V>(uu, b, lp, mp, ff);
        else tet4_product<V>(uu, b, lp, mp, ff);
#endif
        if constexpr (DOTS) edot(uu, ff, [](int a) { return a; }, ma, mb, ma == 0u);
        if (ma == 0u) {  // (branch hoisted out of the row loop: one divergence region, not one per row)
#pragma unroll
          for (int k = 0; k < Geo::NA_OWN; ++k) {
            const int a = Geo::a_own(k);
            T* row = f + static_cast<size_t>(static_cast<uint32_t>(w[a])) * B + col;
#pragma unroll
            for (int c = 0; c < 3; ++c) EXP_RED(reinterpret_cast<V*>(row + c * B), ff[a][c]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < Geo::NA_OWN; ++k) {
            const int a = Geo::a_own(k);
            T* row = f + static_cast<size_t>(static_cast<uint32_t>(w[a])) * B + col;
#pragma unroll
            for (int c = 0; c < 3; ++c) red_p(reinterpret_cast<V*>(row + c * B), ff[a][c], (ma >> (3 * a + c)) & 1u);
          }
        }
#pragma unroll
        for (int k = 0; k < Geo::NFACE; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) carry[k][c] = ff[Geo::a_face(k)][c];
      }
      {  // B (a null B for unpaired A: zero record, own rows masked)
        T rec[12];
        load_rec(cf + 12, rec);
        V b[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) b[k][d] = O::splat(rec[3 * k + d]);
        const V lp = O::splat(rec[9]), mp = O::splat(rec[10]);
        V uu[NPE][3];
#pragma unroll
        for (int a = 0; a < NPE; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) uu[a][c] = dof(src, Geo::b_row(a) * 3 + c);
        V ff[NPE][3];
#if defined(EXP_NOMATH)
        for (int a = 0; a < NPE; ++a) for (int c = 0; c < 3; ++c) ff[a][c] = O::mul(uu[a][c], b[c][c]);
#else
        if constexpr (NPE == 10) tet10_product<V>(uu, b, lp, mp, ff);
        else tet4_product<V>(uu, b, lp, mp, ff);
#endif
        if constexpr (DOTS)
          edot(uu, ff, [](int a) { return Geo::b_row(a); }, ma, mb, ma == 0u && mb == unsigned(kHasB));
#pragma unroll
        for (int k = 0; k < Geo::NFACE; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) ff[Geo::b_face(k)][c] = O::add(ff[Geo::b_face(k)][c], carry[k][c]);
        if (ma == 0u && mb == unsigned(kHasB)) {
#pragma unroll
          for (int a = 0; a < NPE; ++a) {
            T* row = f + static_cast<size_t>(static_cast<uint32_t>(w[Geo::b_row(a)])) * B + col;
#pragma unroll
            for (int c = 0; c < 3; ++c) EXP_RED(reinterpret_cast<V*>(row + c * B), ff[a][c]);
          }
        } else {
#pragma unroll
          for (int a = 0; a < NPE; ++a) {
            const int r = Geo::b_row(a);
            T* row = f + static_cast<size_t>(static_cast<uint32_t>(w[r])) * B + col;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const unsigned m = r < NPE ? (ma >> (3 * r + c)) & 1u : (mb >> (3 * (r - NPE) + c)) & 1u;
              red_p(reinterpret_cast<V*>(row + c * B), ff[a][c], m);
            }
          }
        }
      }
    }
    __syncwarp();
    e = en;
    s ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#if defined(EXP_NORED)
  if (reinterpret_cast<const float*>(&sink)[0] == 1.2345f) f[0] = T(1);
#endif
  if constexpr (DOTS) {  // lane groups folded in order: dpart[block][0][column]
    __shared__ double dred[GROUPS * B];
#pragma unroll
    for (int c = 0; c < CPT; ++c) dred[grp * B + col + c] = dacc[c];
    __syncthreads();
    const int t = threadIdx.x;
    if (t < B) {
      double sum = 0.0;
      for (int g = 0; g < GROUPS; ++g) sum += dred[g * B + t];
      dpart[(int64_t(blockIdx.x) * 3 + 0) * B + t] = sum;
      dpart[(int64_t(blockIdx.x) * 3 + 1) * B + t] = 0.0;
      dpart[(int64_t(blockIdx.x) * 3 + 2) * B + t] = 0.0;
    }
  }
}

// sum over the constrained dofs of p^2 per column (their product rows are the identity, so they
// add p.p to (p, A p)); fixed block ranges and in-block order: reproducible. dpart[block][3][B].
__global__ void __launch_bounds__(256) k_masked_pp(const float* __restrict__ p, const int32_t* __restrict__ dofs,
                                                   int32_t n, int32_t B, double* __restrict__ dpart) {
  __shared__ double sm[256];
  const int t = threadIdx.x, per = 256 / B, col = t % B, slot = t / B;
  double s = 0.0;
  if (slot < per) {
    const int64_t step = int64_t(gridDim.x) * per;
    int64_t i = int64_t(blockIdx.x) * per + slot;
    for (; i + 3 * step < n; i += 4 * step) {  // four independent loads in flight
      int32_t d[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = __ldg(dofs + i + j * step);
      float x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = p[int64_t(d[j]) * B + col];
#pragma unroll
      for (int j = 0; j < 4; ++j) s += double(x[j]) * double(x[j]);
    }
    for (; i < n; i += step) {
      const double x = double(p[int64_t(__ldg(dofs + i)) * B + col]);
      s += x * x;
    }
  }
  sm[t] = slot < per ? s : 0.0;
  __syncthreads();
  if (t < B) {
    double sum = 0.0;
    for (int j = 0; j < per; ++j) sum += sm[j * B + t];
    dpart[(int64_t(blockIdx.x) * 3 + 0) * B + t] = sum;
    dpart[(int64_t(blockIdx.x) * 3 + 1) * B + t] = 0.0;
    dpart[(int64_t(blockIdx.x) * 3 + 2) * B + t] = 0.0;
  }
}

// Units per launch. The persistent grid's lane groups stride through the units
// without synchronising, so over thousands of strides they drift apart and the
// front of concurrently swept elements spreads over the mesh, losing the L2
// reuse of shared node rows. Splitting a long sweep into launches of a bounded
// number of strides re-aligns the front (TSGPU_EBE_PAIR_STRIDES, 0 = one launch).
// configs[3] on one device, fp32 r=8: 29.3 -> 24.6 ms (5300 strides); configs[1] stays one launch (`profiles/r01_pair_strides.txt`).
constexpr int64_t kPairLaunchStrides = 1024;
}  // namespace
bool pair_dynamic() {
  static const bool on = [] {
    const char* e = std::getenv("TSGPU_EBE_DYN");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
int64_t strided_launch_units(int64_t units_per_stride, int64_t units) {
  static const int64_t strides = [] {
    const char* e = std::getenv("TSGPU_EBE_PAIR_STRIDES");
    return e ? std::max<int64_t>(0, std::atoll(e)) : kPairLaunchStrides;
  }();
  if (strides == 0) return std::max<int64_t>(units, 1);
  // equal launches of at most `strides` strides each
  const int64_t cap = strides * units_per_stride, n = (units + cap - 1) / cap;
  return std::max<int64_t>((units + n - 1) / n, 1);
}
int64_t pair_launch_units(int64_t units_per_stride, int64_t units) {
  // the dynamic schedule keeps the front tight by itself: one launch (unless strides are forced)
  if (pair_dynamic() && !std::getenv("TSGPU_EBE_PAIR_STRIDES")) return std::max<int64_t>(units, 1);
  return strided_launch_units(units_per_stride, units);
}
namespace {

template <typename T, typename V, int NPE, int B>
bool launch_pair_b(const ts_ebe& op, const T* u, T* f, cudaStream_t s, int32_t p0, int32_t p1) {
  constexpr int CPT = LaneOps<V>::kCols;
  constexpr int TPE = (B + CPT - 1) / CPT;
  if constexpr (128 % TPE != 0 || TPE * CPT != B) {
    return false;
  } else {
    using Geo = PairGeo<NPE>;
    constexpr int NT = 128, GROUPS = NT / TPE;
    const size_t smem = 2 * (size_t((Geo::NR * 3 + 1) & ~1) * NT * sizeof(V) + size_t(GROUPS) * 24 * sizeof(T) +
                             size_t(GROUPS) * Geo::WORDS * sizeof(int32_t));
    auto kern = k_ebe_pair<T, V, NPE, B, false>;
    const KernelFit fit = kernel_fit<k_ebe_pair<T, V, NPE, B, false>>(NT, smem);
    const int sms = fit.sms, per_sm = std::max(fit.per_sm, 1);
    if (p1 <= p0) return true;
    const int64_t need = (int64_t(p1 - p0) + GROUPS - 1) / GROUPS;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * per_sm)));
    const int64_t step = pair_launch_units(int64_t(grid) * GROUPS, int64_t(p1) - p0);
    for (int64_t a = p0; a < p1; a += step) {
      const int32_t b = static_cast<int32_t>(std::min<int64_t>(p1, a + step));
      int32_t* sched = nullptr;
      if (pair_dynamic()) {
        sched = op.pair->sched.get() + (op.pair->next_slot.fetch_add(1, std::memory_order_relaxed) & 63u);
        TS_CUDA(cudaMemsetAsync(sched, 0, sizeof(int32_t), s));
      }
      kern<<<grid, NT, smem, s>>>(op.pair->conn.get(), reinterpret_cast<const T*>(op.pair->coef.get()),
                                  static_cast<int32_t>(a), b, u, f, sched, nullptr);
      TS_CUDA_LAUNCH();
    }
    return true;
  }
}

// launches of one pair sweep over units [p0, p1) (the split of launch_pair_b); -1 = batch not covered
template <typename T, typename V, int NPE, int B>
int pair_launches_b(int32_t p0, int32_t p1) {
  constexpr int CPT = LaneOps<V>::kCols;
  constexpr int TPE = (B + CPT - 1) / CPT;
  if constexpr (128 % TPE != 0 || TPE * CPT != B) {
    return -1;
  } else {
    using Geo = PairGeo<NPE>;
    constexpr int NT = 128, GROUPS = NT / TPE;
    const size_t smem = 2 * (size_t((Geo::NR * 3 + 1) & ~1) * NT * sizeof(V) + size_t(GROUPS) * 24 * sizeof(T) +
                             size_t(GROUPS) * Geo::WORDS * sizeof(int32_t));
    const KernelFit fit = kernel_fit<k_ebe_pair<T, V, NPE, B, false>>(NT, smem);
    if (p1 <= p0) return 0;
    const int64_t need = (int64_t(p1 - p0) + GROUPS - 1) / GROUPS;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(fit.sms) * std::max(fit.per_sm, 1))));
    const int64_t step = pair_launch_units(int64_t(grid) * GROUPS, int64_t(p1) - p0);
    return static_cast<int>((int64_t(p1) - p0 + step - 1) / step);
  }
}
template <typename T, typename V, int NPE>
int pair_launches_t(int32_t batch, int32_t p0, int32_t p1) {
  switch (batch) {
    case 1: return pair_launches_b<T, T, NPE, 1>(p0, p1);
    case 2: return pair_launches_b<T, V, NPE, 2>(p0, p1);
    case 4: return pair_launches_b<T, V, NPE, 4>(p0, p1);
    case 8: return pair_launches_b<T, V, NPE, 8>(p0, p1);
    case 16: return pair_launches_b<T, V, NPE, 16>(p0, p1);
    default: return -1;
  }
}

template <typename T, typename V, int NPE>
bool launch_pair_t(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int32_t p0, int32_t p1) {
  switch (batch) {
    case 1: return launch_pair_b<T, T, NPE, 1>(op, u, f, s, p0, p1);
    case 2: return launch_pair_b<T, V, NPE, 2>(op, u, f, s, p0, p1);
    case 4: return launch_pair_b<T, V, NPE, 4>(op, u, f, s, p0, p1);
    case 8: return launch_pair_b<T, V, NPE, 8>(op, u, f, s, p0, p1);
    case 16: return launch_pair_b<T, V, NPE, 16>(op, u, f, s, p0, p1);
    default: return false;
  }
}

bool inv3(const double j[3][3], double inv[3][3]) {
  const double d = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) - j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                   j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
  if (d == 0.0) return false;
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
  return true;
}

}  // namespace

constexpr int kPartialRows = 1184;  // blas.h kRedBlocks: rows of the gamma partials workspace
template <int B>
int launch_pair_dots(const ts_ebe& op, const float* u, float* f, cudaStream_t s, double* dpart, int32_t p0,
                     int32_t p1) {
  using T = float;
  using V = float2;
  using Geo = PairGeo<10>;
  constexpr int CPT = LaneOps<V>::kCols, TPE = (B + CPT - 1) / CPT, NT = 128, GROUPS = NT / TPE;
  const size_t smem = 2 * (size_t((Geo::NR * 3 + 1) & ~1) * NT * sizeof(V) + size_t(GROUPS) * 24 * sizeof(T) +
                           size_t(GROUPS) * Geo::WORDS * sizeof(int32_t));
  const KernelFit fit = kernel_fit<k_ebe_pair<T, V, 10, B, true>>(NT, smem);
  if (p1 <= p0) return 0;
  const int64_t need = (int64_t(p1) - p0 + GROUPS - 1) / GROUPS;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(fit.sms) * std::max(fit.per_sm, 1))));
  int32_t* sched = op.pair->sched.get() + (op.pair->next_slot.fetch_add(1, std::memory_order_relaxed) & 63u);
  TS_CUDA(cudaMemsetAsync(sched, 0, sizeof(int32_t), s));
  k_ebe_pair<T, V, 10, B, true><<<grid, NT, smem, s>>>(op.pair->conn.get(), reinterpret_cast<const T*>(op.pair->coef.get()),
                                                       p0, p1, u, f, sched, dpart);
  TS_CUDA_LAUNCH();
  return grid;
}

int ebe_masked_pp(const int32_t* dofs, int32_t n, const float* p, int32_t batch, cudaStream_t s, double* dpart,
                  int rows_left) {
  if (n <= 0 || rows_left <= 0) return 0;
  const int per = 256 / batch;  // dofs per block pass; about 8 passes per thread, within the partial rows left
  const int mb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(rows_left, (int64_t(n) + 8 * per - 1) / (8 * per))));
  k_masked_pp<<<mb, 256, 0, s>>>(p, dofs, n, batch, dpart);
  TS_CUDA_LAUNCH();
  return mb;
}

int ebe_pair_apply_dots(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, double* dpart,
                        int part) {
  static const bool on = [] {  // TSGPU_EBE_FUSED_DOTS=0: the product, then the separate gamma pass
    const char* e = std::getenv("TSGPU_EBE_FUSED_DOTS");
    return !e || e[0] != '0';
  }();
  if (!on || !op.pair || !pair_dynamic() || op.prec != 32 || op.order != 2 || op.deterministic || op.fan) return -1;
  if (batch != 16 && batch != 8) return -1;
  const int32_t U = op.pair->n_units, sp = op.pair->group_split;
  if (part < 0 && sp != 0 && sp != U) return -1;  // the whole sweep in one launch needs one element group
  const int32_t p0 = part == 1 ? sp : 0, p1 = part == 0 ? sp : U;
  const float* uu = static_cast<const float*>(u);
  float* ff = static_cast<float*>(f);
  int nb = batch == 16 ? launch_pair_dots<16>(op, uu, ff, s, dpart, p0, p1) : launch_pair_dots<8>(op, uu, ff, s, dpart, p0, p1);
  if (part < 0 && op.has_mask && op.n_masked_dofs > 0)  // one device: every constrained dof is this rank's
    nb += ebe_masked_pp(op.masked_dofs.get(), op.n_masked_dofs, uu, batch, s, dpart + int64_t(nb) * 3 * batch,
                        kPartialRows - nb);
  return nb;
}

bool ebe_pair_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part) {
  if (!op.pair) return false;
  const int32_t p0 = part == 1 ? op.pair->group_split : 0;
  const int32_t p1 = part == 0 ? op.pair->group_split : op.pair->n_units;
  return ebe_pair_apply_range(op, u, f, batch, s, p0, p1);
}

int ebe_pair_launches(const ts_ebe& op, int32_t batch) {
  if (!op.pair) return -1;
  const int32_t n = op.pair->n_units, sp = op.pair->group_split;
  auto count = [&](int32_t p0, int32_t p1) {
    if (op.prec == 32)
      return op.order == 2 ? pair_launches_t<float, float2, 10>(batch, p0, p1) : pair_launches_t<float, float2, 4>(batch, p0, p1);
    return op.order == 2 ? pair_launches_t<double, double, 10>(batch, p0, p1) : pair_launches_t<double, double, 4>(batch, p0, p1);
  };
  const int a = count(0, sp), b = count(sp, n);
  return a < 0 || b < 0 ? -1 : a + b;
}

bool ebe_unit_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t q0,
                          int32_t q1) {
  if (op.fan) return ebe_fan_apply_range(op, u, f, batch, s, q0, q1);
  return ebe_pair_apply_range(op, u, f, batch, s, q0, q1);
}

int32_t ebe_unit_count(const ts_ebe& op) { return op.fan ? op.fan->n_units : op.pair ? op.pair->n_units : 0; }

bool ebe_pair_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t p0,
                          int32_t p1) {
  if (!op.pair) return false;
  if (op.prec == 32) {
    const float* uu = static_cast<const float*>(u);
    float* ff = static_cast<float*>(f);
    return op.order == 2 ? launch_pair_t<float, float2, 10>(op, uu, ff, batch, s, p0, p1)
                         : launch_pair_t<float, float2, 4>(op, uu, ff, batch, s, p0, p1);
  }
  const double* uu = static_cast<const double*>(u);
  double* ff = static_cast<double*>(f);
  return op.order == 2 ? launch_pair_t<double, double, 10>(op, uu, ff, batch, s, p0, p1)
                       : launch_pair_t<double, double, 4>(op, uu, ff, batch, s, p0, p1);
}

// Pair plan: greedy face matching in (group, Morton) order, then per unit the
// permuted connectivity words (3*node), mask bits and coefficient records.
//   conn_words: Morton-ordered [E][cs] node | mask << 28; coef64: Morton-ordered
//   [E][12] fp64 (b rows, lambda V, mu V, V); vrnd: T-rounded vertex coordinates.
void build_pair_plan(ts_ebe& op, const Mesh& m, const HostVec<int32_t>& conn_words, int cs,
                     const HostVec<double>& coef64, bool fp32, PairTopology* topo) {
  const int npe = op.npe;
  const int NR = npe == 10 ? PairGeo<10>::NR : PairGeo<4>::NR;
  const int kPairWords = npe == 10 ? PairGeo<10>::WORDS : PairGeo<4>::WORDS;
  const int64_t E = op.n_elems;
  static constexpr int ev[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  auto node = [&](int64_t e, int a) { return static_cast<int32_t>(conn_words[e * cs + a] & 0x0FFFFFFF); };
  auto mbits = [&](int64_t e, int a) { return (static_cast<uint32_t>(conn_words[e * cs + a]) >> 28) & 7u; };
  auto edge_slot = [&](int p, int q) {
    for (int k = 0; k < 6; ++k)
      if ((ev[k][0] == p && ev[k][1] == q) || (ev[k][0] == q && ev[k][1] == p)) return 4 + k;
    return -1;
  };
  std::vector<int32_t> mate;
  std::vector<int8_t> mate_k;
  std::vector<int32_t> units;  // leader element; singles encoded as ~e
  int32_t split = 0;
  if (topo && topo->n_elems == E && topo->group_split == op.group_split && !topo->units.empty()) {
    // the level set's other tet10 operator: same mesh, same element order -> same pairs
    mate = topo->mate;
    mate_k = topo->mate_k;
    units = topo->units;
    split = topo->split;
  } else {
    // face adjacency through the vertex -> element incidence: the element across
    // face k (opposite local vertex k) is the other element containing its 3 vertices
    // (parallel counting sort; the order inside a vertex's list does not matter:
    // the element across a face is unique)
    int32_t nv = 0;
#pragma omp parallel for schedule(static) reduction(max : nv)
    for (int64_t e = 0; e < E; ++e)
      for (int a = 0; a < 4; ++a) nv = std::max(nv, node(e, a) + 1);
    std::vector<int32_t> vptr(size_t(nv) + 1, 0);
    HostVec<int32_t> velem(size_t(E) * 4);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
      for (int a = 0; a < 4; ++a) __atomic_fetch_add(&vptr[node(e, a) + 1], 1, __ATOMIC_RELAXED);
    for (int32_t v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
    {
      std::vector<int32_t> cur(vptr.begin(), vptr.end() - 1);
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < 4; ++a)
          velem[__atomic_fetch_add(&cur[node(e, a)], 1, __ATOMIC_RELAXED)] = static_cast<int32_t>(e);
    }
    HostVec<std::array<int32_t, 4>> nbr(E);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
      for (int k = 0; k < 4; ++k) {
        int32_t f3[3], n = 0;
        for (int a = 0; a < 4; ++a)
          if (a != k) f3[n++] = node(e, a);
        int32_t found = -1;
        for (int32_t p = vptr[f3[0]]; p < vptr[f3[0] + 1] && found < 0; ++p) {
          const int32_t j = velem[p];
          if (j == e) continue;
          int hits = 0;
          for (int a = 0; a < 4; ++a) {
            const int32_t x = node(j, a);
            hits += (x == f3[1]) + (x == f3[2]);
          }
          if (hits == 2) found = j;
        }
        nbr[e][k] = found;
      }
    setup_mark("pair: face adjacency");
    auto group_of = [&](int64_t e) { return e < op.group_split ? 0 : 1; };
    mate.assign(E, -1);
    mate_k.assign(E, -1);
    for (int64_t e = 0; e < E; ++e) {
      if (mate[e] >= 0) continue;
      int best = -1;
      int64_t bd = 0;
      for (int k = 0; k < 4; ++k) {
        const int32_t j = nbr[e][k];
        // only later elements: the unit's leader (its lower element) then always carries the face
        // index. On a manifold mesh an unmatched earlier neighbour cannot exist (it would have taken
        // e); on a non-manifold one (a face shared by three elements) the face relation is not
        // symmetric and an earlier j could not name its face towards e.
        if (j < 0 || j <= e || mate[j] >= 0 || group_of(j) != group_of(e)) continue;
        const int64_t d = std::llabs(int64_t(j) - e);
        if (best < 0 || d < bd) {
          best = k;
          bd = d;
        }
      }
      if (best >= 0) {
        const int32_t j = nbr[e][best];
        mate[e] = j;
        mate[j] = static_cast<int32_t>(e);
        mate_k[e] = static_cast<int8_t>(best);
      }
    }
    // units in element order (a pair sits at its lower element, singles in place),
    // so consecutive unit ranges stay spatially compact (ebe_stream.cu chunks them)
    for (int g = 0; g < 2; ++g) {
      const int64_t lo = g == 0 ? 0 : op.group_split, hi = g == 0 ? op.group_split : E;
      for (int64_t e = lo; e < hi; ++e) {
        if (mate[e] > e) units.push_back(static_cast<int32_t>(e));
        else if (mate[e] < 0) units.push_back(~static_cast<int32_t>(e));
      }
      if (g == 0) split = static_cast<int32_t>(units.size());
    }

    if (topo) {
      topo->n_elems = E;
      topo->group_split = op.group_split;
      topo->mate = mate;
      topo->mate_k = mate_k;
      topo->units = units;
      topo->split = split;
    }
  }
  setup_mark("pair: matching");
  const int32_t U = static_cast<int32_t>(units.size());
  HostVec<int32_t> pc(size_t(U) * kPairWords);
  const size_t ts = fp32 ? 4 : 8;
  HostVec<unsigned char> pcf(size_t(U) * 24 * ts);
  auto rnd = [fp32](double x) { return fp32 ? static_cast<double>(static_cast<float>(x)) : x; };
  // coefficient record of element e with local vertex order perm (orientation from the original order)
  auto record = [&](int64_t e, const int perm[4], unsigned char* dst) -> bool {
    double v[4][3], j[3][3], inv[3][3];
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 3; ++c) v[a][c] = rnd(m.coords[3 * size_t(op.host_conn[e * npe + perm[a]]) + c]);
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) j[r][c] = v[c + 1][r] - v[0][r];
    if (!inv3(j, inv)) return false;
    double rec[12];
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) rec[3 * k + d] = inv[k][d];
    const double scale = npe == 10 ? 1.0 / 20.0 : 1.0;
    rec[9] = coef64[12 * e + 9] * scale;   // lambda V (/ 20 for tet10), original orientation
    rec[10] = coef64[12 * e + 10] * scale; // mu V
    rec[11] = 0.0;
    for (int q = 0; q < 12; ++q) {
      if (fp32) {
        const float x = static_cast<float>(rec[q]);
        std::memcpy(dst + q * 4, &x, 4);
      } else {
        std::memcpy(dst + q * 8, &rec[q], 8);
      }
    }
    return true;
  };
  auto slot_node = [&](int64_t e, const int perm[4], int s) -> std::pair<int32_t, uint32_t> {
    const int a = s < 4 ? perm[s] : edge_slot(perm[ev[s - 4][0]], perm[ev[s - 4][1]]);
    return {node(e, a), mbits(e, a)};
  };
  bool bad = false;
#pragma omp parallel for schedule(static) reduction(|| : bad)
  for (int32_t i = 0; i < U; ++i) {
    int32_t* w = pc.data() + size_t(i) * kPairWords;
    unsigned char* cf = pcf.data() + size_t(i) * 24 * ts;
    const bool single = units[i] < 0;
    const int64_t a = single ? ~units[i] : units[i];
    int pa[4] = {0, 1, 2, 3};
    uint32_t ma = 0, mb = 0;
    if (!single) {
      const int k = mate_k[a];
      const int64_t b = mate[a];
      // A: (opposite vertex k, then the face vertices in A's order); B: the face vertices in A's order, then its 4th
      int n = 1;
      pa[0] = k;
      for (int q = 0; q < 4; ++q)
        if (q != k) pa[n++] = q;
      int pb[4];
      for (int q = 1; q < 4; ++q) {
        pb[q - 1] = -1;
        for (int r = 0; r < 4; ++r)
          if (node(b, r) == node(a, pa[q])) pb[q - 1] = r;
        if (pb[q - 1] < 0) bad = true;
      }
      if (pb[0] < 0 || pb[1] < 0 || pb[2] < 0) continue;
      for (int r = 0; r < 4; ++r)
        if (r != pb[0] && r != pb[1] && r != pb[2]) pb[3] = r;
      for (int s = 0; s < npe; ++s) {
        const auto [nd, mk] = slot_node(a, pa, s);
        w[s] = 3 * nd;
        ma |= mk << (3 * s);
      }
      const int nbown = NR - npe;
      for (int q = 0; q < nbown; ++q) {
        const int sl = npe == 10 ? PairGeo<10>::b_own(q) : PairGeo<4>::b_own(q);
        const auto [nd, mk] = slot_node(b, pb, sl);
        w[npe + q] = 3 * nd;
        mb |= mk << (3 * q);
      }
      // the shared face: B's face slots are A's face slots
      const int nface = npe == 10 ? PairGeo<10>::NFACE : PairGeo<4>::NFACE;
      for (int q = 0; q < nface; ++q) {
        const int bs = npe == 10 ? PairGeo<10>::b_face(q) : PairGeo<4>::b_face(q);
        const int as = npe == 10 ? PairGeo<10>::a_face(q) : PairGeo<4>::a_face(q);
        if (slot_node(b, pb, bs).first * 3 != w[as]) bad = true;
      }
      bad = bad || !record(a, pa, cf) || !record(b, pb, cf + 12 * ts);
    } else {
      for (int s = 0; s < npe; ++s) {
        const auto [nd, mk] = slot_node(a, pa, s);
        w[s] = 3 * nd;
        ma |= mk << (3 * s);
      }
      // no face neighbour: a pair with a NULL B (zero record, own rows fully masked -> no gather, no
      // reduction), so every unit takes the same code path; its face rows reduce through B's
      for (int s = npe; s < NR; ++s) w[s] = 0;
      std::memset(cf + 12 * ts, 0, 12 * ts);
      mb = (1u << (3 * (NR - npe))) - 1u;
      bad = bad || !record(a, pa, cf);
    }
    w[NR] = static_cast<int32_t>(ma);
    w[NR + 1] = static_cast<int32_t>(mb | uint32_t(kHasB));
    for (int s = NR + 2; s < kPairWords; ++s) w[s] = 0;
  }
  if (bad) validation("pair plan: inconsistent face pairing or degenerate element");
  setup_mark("pair: unit records");
  auto plan = std::make_unique<EbePairPlan>();
  plan->n_units = U;
  plan->group_split = split;
  int64_t paired = 0;
  for (int32_t x : units) paired += x >= 0 ? 2 : 0;
  plan->paired_fraction = E ? double(paired) / double(E) : 0.0;
  plan->conn.upload(pc);
  plan->coef.upload(pcf);
  plan->sched.alloc(64);
  op.pair = std::move(plan);
}

}  // namespace tsg
