// ebe_fan.cu — EBE sweep over EDGE FANS of tet10 elements.
//
// Same product as the pair sweep (ebe_operator.hpp:143-188 semantics, the lean
// exact element math of element_kernels.cuh); what changes is the unit of work.
// A fan is a run of elements around one mesh edge (p, q): element j of a fan is
// (p, q, r_j, r_{j+1}), consecutive elements share the face (p, q, r_{j+1}),
// and a closed fan comes back to r_0 (the ring around an interior edge; the six
// Kuhn tets of a box cell around its diagonal). Labelling every element of a
// fan (p, q, r_j, r_{j+1}) — a relabelling of its local vertices; gradients in
// the new order, volume from the original orientation, so K_e is unchanged —
// puts the rows a fan's consecutive elements share in fixed register roles:
//   p, q, m = mid(p, q)            in every element       (accumulated, reduced at the end)
//   r_j, mid(p, r_j), mid(q, r_j)  in elements j-1 and j  (carried one step, then reduced)
//   mid(r_j, r_{j+1})              in element j only      (reduced at once)
// so a fan of k elements gathers and scatter-adds 4k + 3 (closed) / 4k + 6
// (open) node rows instead of 10k (singles) or 7k (face pairs): a closed 6-fan
// moves 4.5 rows per element. The memory path alone (scripts/micro/unit_paths.cu,
// configs[1], r = 16 fp32): singles 1.14 ms, pairs 0.81 ms, 6-fans 0.61 ms.
//
// A lane group (TPE lanes x CPT cases = the batch) walks its fans element by
// element; while it computes element t, the rows element t+1 adds (4 rows: the
// next ring vertex's 3 rows and the next ring edge; 10 at a fan's start) and
// element t+1's coefficient record stream into shared memory (cp.async), as do
// the row words of element t+2. Row slots per group: two fan headers (p, q, m,
// r_0 rows; alternating between consecutive fans), three ring-vertex triples
// (rotating), two ring edges (alternating), and r_0's partial sums of a closed
// fan (parked in shared memory between its first and last element).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {
namespace {

// element word record: 12 int32 = [flags, gathered rows g1 .. g10, 0]; a row word is
// node | dof-mask bits << 28 (bare node ids when the element has no constrained dof: the
// kInterior fast paths). The rows an element scatter-adds are the ones gathered before it
// (A: the previous element's B; at a fan's end, B and p, q, m), carried in registers.
enum : int32_t { kFanStart = 1, kFanEnd = 2, kFanClosed = 4, kFanInterior = 8 };
constexpr int kFanWords = 12;
constexpr int kHdrSlots = 6;                    // p, q, m, r0, mid(p,r0), mid(q,r0)
constexpr int kRingBase = 2 * kHdrSlots;        // 3 ring-vertex triples
constexpr int kEdgeBase = kRingBase + 9;        // 2 ring edges
constexpr int kR0Base = kEdgeBase + 2;          // r0 partial sums of a closed fan
constexpr int kFanSlots = kR0Base + 3;          // row slots per lane group
constexpr int kRowV = 4;                        // lane vectors per row slot (3 components + pad)

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

// one lane's 3 components of a row slot (16-byte shared loads)
template <typename V>
__device__ __forceinline__ void load_row(const V* p, V (&r)[3]) {
  if constexpr (sizeof(V) == 8) {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0];
    const uint2 b = reinterpret_cast<const uint2*>(p)[2];
    r[0] = *reinterpret_cast<const V*>(&a.x);
    r[1] = *reinterpret_cast<const V*>(&a.z);
    r[2] = *reinterpret_cast<const V*>(&b.x);
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p);
    r[0] = a.x; r[1] = a.y; r[2] = a.z;
  }
}
template <typename V>
__device__ __forceinline__ void store_row(V* p, const V (&r)[3]) {
  p[0] = r[0]; p[1] = r[1]; p[2] = r[2];
}

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

// The group's element stream: its fans u = first, first + G, ... in [.., u1), each
// [ufirst[u], ufirst[u+1]); the next fan's bounds are loaded one fan ahead.
struct FanCursor {
  int32_t x = -1, end = 0, un = 0, nf = 0, ne = 0;
  __device__ __forceinline__ void prefetch(const int32_t* __restrict__ uf, int32_t u1, int32_t G) {
    if (un + G < u1) {
      nf = __ldg(uf + un + G);
      ne = __ldg(uf + un + G + 1);
    }
  }
  __device__ __forceinline__ void init(const int32_t* __restrict__ uf, int32_t u, int32_t u1, int32_t G) {
    un = u;
    if (u < u1) {
      x = __ldg(uf + u);
      end = __ldg(uf + u + 1);
      prefetch(uf, u1, G);
    } else {
      x = -1;
    }
  }
  __device__ __forceinline__ void advance(const int32_t* __restrict__ uf, int32_t u1, int32_t G) {
    if (x < 0) return;
    if (++x == end) {
      un += G;
      if (un < u1) {
        x = nf;
        end = ne;
        prefetch(uf, u1, G);
      } else {
        x = -1;
      }
    }
  }
};

template <typename T, typename V, int B>
__global__ void __launch_bounds__(128, 2)
k_ebe_fan(const int4* __restrict__ words, const T* __restrict__ coef, const int32_t* __restrict__ ufirst,
          int32_t u0, int32_t u1, const T* __restrict__ u, T* __restrict__ f) {
  using O = LaneOps<V>;
  constexpr int CPT = O::kCols;
  constexpr int TPE = (B + CPT - 1) / CPT;
  constexpr int NT = 128;
  static_assert(NT % TPE == 0 && TPE * CPT == B, "lane groups must tile the block and the batch");
  constexpr int GROUPS = NT / TPE;
  constexpr int TPC = 16 / sizeof(T);
  constexpr int RCH = 12 / TPC;   // 16-byte chunks per coefficient record
  constexpr int RS = TPE * kRowV; // lane vectors per row slot
  extern __shared__ __align__(16) unsigned char smem[];
  const int grp = threadIdx.x / TPE;
  const int lane = threadIdx.x % TPE;
  V* const ug = reinterpret_cast<V*>(smem) + size_t(grp) * kFanSlots * RS + lane * kRowV;  // this lane's slot 0
  T* const cg = reinterpret_cast<T*>(smem + size_t(NT) * kFanSlots * kRowV * sizeof(V)) + size_t(grp) * 24;
  int4* const wg =
      reinterpret_cast<int4*>(smem + size_t(NT) * kFanSlots * kRowV * sizeof(V) + size_t(GROUPS) * 24 * sizeof(T)) +
      size_t(grp) * 9;
  const int col = lane * CPT;
  const T* const ub = u + col;
  T* const fb = f + col;
  const int32_t G = gridDim.x * GROUPS;

  // rows: interior elements carry bare node ids (no mask bits), so one IMAD addresses a row
  auto gather_plain = [&](int32_t w, V* dst) {
    const T* src = ub + static_cast<size_t>(static_cast<uint32_t>(w)) * (3 * B);
#pragma unroll
    for (int c = 0; c < 3; ++c) cpa(dst + c, src + c * B, int(sizeof(V)), sizeof(V));
  };
  auto gather_mask = [&](int32_t w, V* dst) {
    const T* src = ub + static_cast<size_t>(static_cast<uint32_t>(w) & 0x0FFFFFFFu) * (3 * B);
    const unsigned mk = static_cast<unsigned>(w) >> 28;
#pragma unroll
    for (int c = 0; c < 3; ++c) cpa(dst + c, src + c * B, ((mk >> c) & 1u) ? 0 : int(sizeof(V)), sizeof(V));
  };
  auto red_plain = [&](int32_t w, const V& a, const V& b, const V& c2) {
    T* dst = fb + static_cast<size_t>(static_cast<uint32_t>(w)) * (3 * B);
    red_lane(reinterpret_cast<V*>(dst), a);
    red_lane(reinterpret_cast<V*>(dst + B), b);
    red_lane(reinterpret_cast<V*>(dst + 2 * B), c2);
  };
  auto red_mask = [&](int32_t w, const V& a, const V& b, const V& c2) {
    T* dst = fb + static_cast<size_t>(static_cast<uint32_t>(w) & 0x0FFFFFFFu) * (3 * B);
    const unsigned mk = static_cast<unsigned>(w) >> 28;
    red_p(reinterpret_cast<V*>(dst), a, mk & 1u);
    red_p(reinterpret_cast<V*>(dst + B), b, (mk >> 1) & 1u);
    red_p(reinterpret_cast<V*>(dst + 2 * B), c2, (mk >> 2) & 1u);
  };
  auto fetch_words = [&](int32_t x, int ws) {
    if (x >= 0)
      for (int q = lane; q < 3; q += TPE) cpa(wg + 3 * ws + q, words + 3 * static_cast<size_t>(x) + q, 16, 16);
  };

  // slot state: of the element whose rows are in flight (n) and of the one computed (c)
  int ring_next = 0, edge_next = 0, hdr_n = 1, bslot_n = -1, eslot_n = 0;
  auto issue = [&](int32_t xn, int wsn, int rsn) {
    if (xn < 0) return;
    const int4* w = wg + 3 * wsn;
    const int4 w0 = w[0], w1 = w[1];
    const int32_t fl = w0.x;
    for (int q = lane; q < RCH; q += TPE) cpa(cg + 12 * rsn + q * TPC, coef + 12 * static_cast<size_t>(xn) + q * TPC, 16, 16);
    if (fl & kFanStart) {
      const int4 w2 = w[2];
      hdr_n ^= 1;
      bslot_n = ring_next;
      ring_next = ring_next == 2 ? 0 : ring_next + 1;
      eslot_n = edge_next;
      edge_next ^= 1;
      V* h = ug + hdr_n * (kHdrSlots * RS);
      V* rb = ug + (kRingBase + 3 * bslot_n) * RS;
      V* eb = ug + (kEdgeBase + eslot_n) * RS;
      if (fl & kFanInterior) {
        gather_plain(w0.y, h);
        gather_plain(w0.z, h + RS);
        gather_plain(w0.w, h + 2 * RS);
        gather_plain(w1.x, h + 3 * RS);
        gather_plain(w1.y, h + 4 * RS);
        gather_plain(w1.z, h + 5 * RS);
        gather_plain(w1.w, rb);
        gather_plain(w2.x, rb + RS);
        gather_plain(w2.y, rb + 2 * RS);
        gather_plain(w2.z, eb);
      } else {
        gather_mask(w0.y, h);
        gather_mask(w0.z, h + RS);
        gather_mask(w0.w, h + 2 * RS);
        gather_mask(w1.x, h + 3 * RS);
        gather_mask(w1.y, h + 4 * RS);
        gather_mask(w1.z, h + 5 * RS);
        gather_mask(w1.w, rb);
        gather_mask(w2.x, rb + RS);
        gather_mask(w2.y, rb + 2 * RS);
        gather_mask(w2.z, eb);
      }
    } else {
      const bool ring = (fl & (kFanEnd | kFanClosed)) != (kFanEnd | kFanClosed);  // else B = r0, in the header
      bslot_n = -1;
      if (ring) {
        bslot_n = ring_next;
        ring_next = ring_next == 2 ? 0 : ring_next + 1;
      }
      eslot_n = edge_next;
      edge_next ^= 1;
      V* rb = ug + (kRingBase + 3 * bslot_n) * RS;
      V* eb = ug + (kEdgeBase + eslot_n) * RS;
      if (fl & kFanInterior) {
        if (ring) {
          gather_plain(w0.y, rb);
          gather_plain(w0.z, rb + RS);
          gather_plain(w0.w, rb + 2 * RS);
        }
        gather_plain(w1.x, eb);
      } else {
        if (ring) {
          gather_mask(w0.y, rb);
          gather_mask(w0.z, rb + RS);
          gather_mask(w0.w, rb + 2 * RS);
        }
        gather_mask(w1.x, eb);
      }
    }
  };

  FanCursor cur;
  cur.init(ufirst, u0 + static_cast<int32_t>(blockIdx.x) * GROUPS + grp, u1, G);
  int32_t xn = cur.x;
  cur.advance(ufirst, u1, G);
  // prologue: words of the first element, then its rows + the second element's words
  fetch_words(xn, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  issue(xn, 0, 0);
  fetch_words(cur.x, 1);
  asm volatile("cp.async.commit_group;" ::: "memory");

  int wsc = 0, rsc = 0;  // word slot (mod 3) and record slot (mod 2) of the computed element
  int aslot = -1;        // ring slot of A (-1: r0 in the header)
  int32_t hw[6] = {0, 0, 0, 0, 0, 0}, aw[3] = {0, 0, 0}, bw[3] = {0, 0, 0};  // p q m r0 rows; A, B rows
  V S[3][3], X[3][3], Y[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) S[i][c] = X[i][c] = Y[i][c] = O::zero();

  // one element; FA holds the A rows' partial sums (in: from the previous element,
  // out: complete), FB receives the B rows (the next element's FA). Two calls per
  // loop trip with the roles swapped keep the carry in place (no register moves).
  auto step = [&](V (&FA)[3][3], V (&FB)[3][3]) -> bool {
    if (!__any_sync(0xffffffffu, xn >= 0)) return false;
    const int32_t xc = xn;
    const int hdr_c = hdr_n, bslot_c = bslot_n, eslot_c = eslot_n;
    xn = cur.x;
    cur.advance(ufirst, u1, G);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const int wsn = wsc == 2 ? 0 : wsc + 1, ws2 = wsn == 2 ? 0 : wsn + 1;
    issue(xn, wsn, rsc ^ 1);
    fetch_words(cur.x, ws2);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (xc >= 0) {
      const int4* w = wg + 3 * wsc;
      const int4 w0 = w[0], w1 = w[1];
      const int32_t fl = w0.x;
      const bool start = (fl & kFanStart) != 0;
      int32_t ew;
      if (start) {
        const int4 w2 = w[2];
        hw[0] = w0.y; hw[1] = w0.z; hw[2] = w0.w; hw[3] = w1.x; hw[4] = w1.y; hw[5] = w1.z;
        aw[0] = w1.x; aw[1] = w1.y; aw[2] = w1.z;
        bw[0] = w1.w; bw[1] = w2.x; bw[2] = w2.y;
        ew = w2.z;
      } else {
        aw[0] = bw[0]; aw[1] = bw[1]; aw[2] = bw[2];
        if (bslot_c < 0) {
          bw[0] = hw[3]; bw[1] = hw[4]; bw[2] = hw[5];
        } else {
          bw[0] = w0.y; bw[1] = w0.z; bw[2] = w0.w;
        }
        ew = w1.x;
      }
      T rec[12];
      load_rec(cg + 12 * rsc, rec);
      V b[3][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) b[k][d] = O::splat(rec[3 * k + d]);
      const V lp = O::splat(rec[9]), mp = O::splat(rec[10]);
      const V* h = ug + hdr_c * (kHdrSlots * RS);
      const V* ra = start ? h + 3 * RS : ug + (kRingBase + 3 * aslot) * RS;
      const V* rb = bslot_c < 0 ? h + 3 * RS : ug + (kRingBase + 3 * bslot_c) * RS;
      V uu[10][3];
      load_row(h, uu[0]);
      load_row(h + RS, uu[1]);
      load_row(h + 2 * RS, uu[4]);
      load_row(ra, uu[2]);
      load_row(ra + RS, uu[6]);
      load_row(ra + 2 * RS, uu[5]);
      load_row(rb, uu[3]);
      load_row(rb + RS, uu[7]);
      load_row(rb + 2 * RS, uu[8]);
      load_row(ug + (kEdgeBase + eslot_c) * RS, uu[9]);
      V FE[3];
      // slots: 0 p, 1 q, 4 m (S) | 2 r_j, 6 mid(p,r_j), 5 mid(q,r_j) (A) | 3, 7, 8 (B) | 9 ring edge
      tet10_product_acc<0x077u>(uu, b, lp, mp, [&](int s, int c) -> V& {
        return s == 0 ? S[0][c] : s == 1 ? S[1][c] : s == 4 ? S[2][c] : s == 2 ? FA[0][c] : s == 6 ? FA[1][c]
             : s == 5 ? FA[2][c] : s == 3 ? FB[0][c] : s == 7 ? FB[1][c] : s == 8 ? FB[2][c] : FE[c];
      });
      const bool end = (fl & kFanEnd) != 0, closed = (fl & kFanClosed) != 0;
      V* const r0park = ug + kR0Base * RS;
      if (start && closed) {  // r_0 of a closed fan: parked until the fan's last element
#pragma unroll
        for (int i = 0; i < 3; ++i) store_row(r0park + i * RS, FA[i]);
      }
      if (end && closed) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          V r[3];
          load_row(r0park + i * RS, r);
#pragma unroll
          for (int c = 0; c < 3; ++c) FB[i][c] = O::add(FB[i][c], r[c]);
        }
      }
      const bool reda = !(start && closed);
      if (fl & kFanInterior) {
        if (reda)
#pragma unroll
          for (int i = 0; i < 3; ++i) red_plain(aw[i], FA[i][0], FA[i][1], FA[i][2]);
        red_plain(ew, FE[0], FE[1], FE[2]);
        if (end) {
#pragma unroll
          for (int i = 0; i < 3; ++i) red_plain(bw[i], FB[i][0], FB[i][1], FB[i][2]);
#pragma unroll
          for (int i = 0; i < 3; ++i) red_plain(hw[i], S[i][0], S[i][1], S[i][2]);
        }
      } else {
        if (reda)
#pragma unroll
          for (int i = 0; i < 3; ++i) red_mask(aw[i], FA[i][0], FA[i][1], FA[i][2]);
        red_mask(ew, FE[0], FE[1], FE[2]);
        if (end) {
#pragma unroll
          for (int i = 0; i < 3; ++i) red_mask(bw[i], FB[i][0], FB[i][1], FB[i][2]);
#pragma unroll
          for (int i = 0; i < 3; ++i) red_mask(hw[i], S[i][0], S[i][1], S[i][2]);
        }
      }
      if (end) {  // the next fan starts from zero partial sums (S, and its A = this B)
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int c = 0; c < 3; ++c) S[i][c] = FB[i][c] = O::zero();
      }
      aslot = bslot_c;
    }
    __syncwarp();
    wsc = wsn;
    rsc ^= 1;
    return true;
  };
  while (step(X, Y) && step(Y, X)) {
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <typename T, typename V, int B>
size_t fan_smem() {
  constexpr int CPT = LaneOps<V>::kCols, TPE = (B + CPT - 1) / CPT, NT = 128, GROUPS = NT / TPE;
  return size_t(NT) * kFanSlots * kRowV * sizeof(V) + size_t(GROUPS) * 24 * sizeof(T) + size_t(GROUPS) * 9 * 16;
}

template <typename T, typename V, int B>
bool launch_fan_b(const ts_ebe& op, const T* u, T* f, cudaStream_t s, int32_t q0, int32_t q1, int* launches) {
  constexpr int CPT = LaneOps<V>::kCols;
  constexpr int TPE = (B + CPT - 1) / CPT;
  if constexpr (128 % TPE != 0 || TPE * CPT != B) {
    return false;
  } else {
    constexpr int NT = 128, GROUPS = NT / TPE;
    const size_t smem = fan_smem<T, V, B>();
    const KernelFit fit = kernel_fit<k_ebe_fan<T, V, B>>(NT, smem);
    if (q1 <= q0) return true;
    const int64_t need = (int64_t(q1 - q0) + GROUPS - 1) / GROUPS;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(fit.sms) * std::max(fit.per_sm, 1))));
    const int64_t step = pair_launch_units(int64_t(grid) * GROUPS, int64_t(q1) - q0);
    for (int64_t a = q0; a < q1; a += step) {
      const int32_t b = static_cast<int32_t>(std::min<int64_t>(q1, a + step));
      if (launches) {
        ++*launches;
        continue;
      }
      k_ebe_fan<T, V, B><<<grid, NT, smem, s>>>(reinterpret_cast<const int4*>(op.fan->words.get()),
                                                reinterpret_cast<const T*>(op.fan->coef.get()), op.fan->ufirst.get(),
                                                static_cast<int32_t>(a), b, u, f);
      TS_CUDA_LAUNCH();
    }
    return true;
  }
}

template <typename T, typename V>
bool launch_fan_t(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int32_t q0, int32_t q1,
                  int* launches) {
  switch (batch) {
    case 1: return launch_fan_b<T, T, 1>(op, u, f, s, q0, q1, launches);
    case 2: return launch_fan_b<T, V, 2>(op, u, f, s, q0, q1, launches);
    case 4: return launch_fan_b<T, V, 4>(op, u, f, s, q0, q1, launches);
    case 8: return launch_fan_b<T, V, 8>(op, u, f, s, q0, q1, launches);
    case 16: return launch_fan_b<T, V, 16>(op, u, f, s, q0, q1, launches);
    default: return false;
  }
}

bool fan_dispatch(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t q0, int32_t q1,
                  int* launches) {
  if (!op.fan) return false;
  if (op.prec == 32)
    return launch_fan_t<float, float2>(op, static_cast<const float*>(u), static_cast<float*>(f), batch, s, q0, q1,
                                       launches);
  return launch_fan_t<double, double>(op, static_cast<const double*>(u), static_cast<double*>(f), batch, s, q0, q1,
                                      launches);
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

bool ebe_fan_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t q0,
                         int32_t q1) {
  return fan_dispatch(op, u, f, batch, s, q0, q1, nullptr);
}

bool ebe_fan_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part) {
  if (!op.fan) return false;
  const int32_t q0 = part == 1 ? op.fan->group_split : 0;
  const int32_t q1 = part == 0 ? op.fan->group_split : op.fan->n_units;
  return fan_dispatch(op, u, f, batch, s, q0, q1, nullptr);
}

int ebe_fan_launches(const ts_ebe& op, int32_t batch) {
  if (!op.fan) return -1;
  int n = 0;
  const int32_t sp = op.fan->group_split, U = op.fan->n_units;
  if (!fan_dispatch(op, nullptr, nullptr, batch, nullptr, 0, sp, &n)) return -1;
  fan_dispatch(op, nullptr, nullptr, batch, nullptr, sp, U, &n);
  return n;
}

// Fan cover (setup, host): elements in sweep order; each unassigned element
// takes the longest run of unassigned same-group elements around one of its six
// edges (closed rings first, then length, then the smallest spread of sweep
// positions, which keeps a box cell's six Kuhn tets together around the cell
// diagonal). Fans are emitted in the order they are formed, so the fan order
// follows the sweep order (slab-major Morton).
void build_fan_plan(ts_ebe& op, const Mesh& m, const HostVec<int32_t>& conn_words, int cs,
                    const HostVec<double>& coef64, bool fp32) {
  if (op.npe != 10) return;
  const int64_t E = op.n_elems;
  const int32_t N = op.n_nodes;
  static constexpr int ev[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  auto node = [&](int64_t e, int a) { return static_cast<int32_t>(conn_words[e * cs + a] & 0x0FFFFFFF); };
  auto word = [&](int64_t e, int a) { return conn_words[e * cs + a]; };
  auto group_of = [&](int64_t e) { return e < op.group_split ? 0 : 1; };
  auto edge_slot = [&](int p, int q) {
    for (int k = 0; k < 6; ++k)
      if ((ev[k][0] == p && ev[k][1] == q) || (ev[k][0] == q && ev[k][1] == p)) return 4 + k;
    return -1;
  };
  // edge-node -> (element, local edge) incidence (counting sort; edge nodes are unique per edge)
  std::vector<int32_t> eptr(size_t(N) + 1, 0);
  HostVec<int32_t> einc(size_t(E) * 6);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e)
    for (int q = 0; q < 6; ++q) __atomic_fetch_add(&eptr[node(e, 4 + q) + 1], 1, __ATOMIC_RELAXED);
  for (int32_t n = 0; n < N; ++n) eptr[n + 1] += eptr[n];
  {
    std::vector<int32_t> cur(eptr.begin(), eptr.end() - 1);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
      for (int q = 0; q < 6; ++q)
        einc[__atomic_fetch_add(&cur[node(e, 4 + q)], 1, __ATOMIC_RELAXED)] = static_cast<int32_t>(e * 8 + q);
  }
  setup_mark("fan: edge incidence");

  std::vector<uint8_t> taken(E, 0);
  std::vector<int32_t> order;  // elements in fan order
  order.reserve(E);
  struct Fan {
    int32_t first;  // into order
    int32_t k;
    bool closed;
    int32_t p, q;   // edge vertices (global node ids)
  };
  std::vector<Fan> fans;
  std::vector<int32_t> ring;         // fan candidates of one edge
  std::vector<std::array<int32_t, 2>> oth;
  std::vector<int32_t> path, best_path;
  for (int64_t e0 = 0; e0 < E; ++e0) {
    if (taken[e0]) continue;
    const int g = group_of(e0);
    int best_k = -1;
    bool best_closed = false;
    int64_t best_span = 0;
    int32_t best_p = 0, best_q = 0;
    for (int qe = 0; qe < 6; ++qe) {
      const int32_t a = node(e0, ev[qe][0]), b = node(e0, ev[qe][1]);
      const int32_t en = node(e0, 4 + qe);
      ring.clear();
      oth.clear();
      for (int32_t t = eptr[en]; t < eptr[en + 1]; ++t) {
        const int32_t e = einc[t] >> 3;
        if (taken[e] || group_of(e) != g) continue;
        std::array<int32_t, 2> o{-1, -1};
        int no = 0;
        for (int v = 0; v < 4; ++v) {
          const int32_t x = node(e, v);
          if (x != a && x != b && no < 2) o[no++] = x;
        }
        if (no != 2) continue;
        ring.push_back(e);
        oth.push_back(o);
      }
      // walk the run through e0: neighbours share one of their two other vertices
      const int nr = static_cast<int>(ring.size());
      int i0 = -1;
      for (int i = 0; i < nr; ++i)
        if (ring[i] == e0) i0 = i;
      if (i0 < 0) continue;
      auto nbr_via = [&](int i, int32_t v, int not_i) {
        for (int j = 0; j < nr; ++j)
          if (j != i && j != not_i && (oth[j][0] == v || oth[j][1] == v)) return j;
        return -1;
      };
      // forward from e0 through oth[i0][1], backward through oth[i0][0]
      std::vector<int> fwd, bwd;
      bool closed = false;
      {
        int prev = i0, cur = i0;
        int32_t v = oth[i0][1];
        while (true) {
          const int nx = nbr_via(cur, v, prev);
          if (nx < 0) break;
          if (nx == i0) {
            closed = true;
            break;
          }
          if (static_cast<int>(fwd.size()) > nr) break;
          fwd.push_back(nx);
          v = oth[nx][0] == v ? oth[nx][1] : oth[nx][0];
          prev = cur;
          cur = nx;
        }
      }
      if (!closed) {
        int prev = i0, cur = i0;
        int32_t v = oth[i0][0];
        while (true) {
          const int nx = nbr_via(cur, v, prev);
          if (nx < 0 || nx == i0) break;
          if (static_cast<int>(bwd.size()) > nr) break;
          bwd.push_back(nx);
          v = oth[nx][0] == v ? oth[nx][1] : oth[nx][0];
          prev = cur;
          cur = nx;
        }
      }
      path.clear();
      for (auto it = bwd.rbegin(); it != bwd.rend(); ++it) path.push_back(ring[*it]);
      path.push_back(e0);
      for (int i : fwd) path.push_back(ring[i]);
      const int k = static_cast<int>(path.size());
      if (closed && k < 3) closed = false;
      int64_t lo = E, hi = -1;
      for (int32_t e : path) {
        lo = std::min<int64_t>(lo, e);
        hi = std::max<int64_t>(hi, e);
      }
      const int64_t span = hi - lo;
      const bool better = best_k < 0 || (closed && !best_closed) ||
                          (closed == best_closed && (k > best_k || (k == best_k && span < best_span)));
      if (better) {
        best_k = k;
        best_closed = closed;
        best_span = span;
        best_path = path;
        best_p = a;
        best_q = b;
      }
    }
    if (best_k < 0) {  // isolated (cannot happen for a valid tet10 element): a fan of one
      best_path.assign(1, static_cast<int32_t>(e0));
      best_k = 1;
      best_closed = false;
      best_p = node(e0, 0);
      best_q = node(e0, 1);
    }
    Fan fn{static_cast<int32_t>(order.size()), best_k, best_closed, best_p, best_q};
    for (int32_t e : best_path) {
      taken[e] = 1;
      order.push_back(e);
    }
    fans.push_back(fn);
  }
  setup_mark("fan: cover");
  const int32_t U = static_cast<int32_t>(fans.size());
  int32_t split = 0;
  for (int32_t i = 0; i < U; ++i)
    if (group_of(order[fans[i].first]) == 0) split = i + 1;

  const size_t ts = fp32 ? 4 : 8;
  HostVec<int32_t> wv(size_t(E) * kFanWords);
  HostVec<unsigned char> cf(size_t(E) * 12 * ts);
  auto rnd = [fp32](double x) { return fp32 ? static_cast<double>(static_cast<float>(x)) : x; };
  bool bad = false;
#pragma omp parallel for schedule(dynamic, 1024) reduction(|| : bad)
  for (int32_t fi = 0; fi < U; ++fi) {
    const Fan& fn = fans[fi];
    const int k = fn.k;
    // ring vertices r_0 .. r_k of the ordered path
    std::vector<int32_t> r(k + 1, -1);
    auto others = [&](int64_t e, int32_t* o) {
      int no = 0;
      for (int v = 0; v < 4; ++v) {
        const int32_t x = node(e, v);
        if (x != fn.p && x != fn.q && no < 2) o[no++] = x;
      }
      return no == 2;
    };
    int32_t o0[2];
    if (!others(order[fn.first], o0)) {
      bad = true;
      continue;
    }
    if (k == 1) {
      r[0] = o0[0];
      r[1] = o0[1];
    } else {
      int32_t o1[2];
      if (!others(order[fn.first + 1], o1)) {
        bad = true;
        continue;
      }
      r[1] = (o0[0] == o1[0] || o0[0] == o1[1]) ? o0[0] : o0[1];
      r[0] = r[1] == o0[0] ? o0[1] : o0[0];
      for (int j = 1; j < k; ++j) {
        int32_t oj[2];
        if (!others(order[fn.first + j], oj)) {
          bad = true;
          break;
        }
        if (oj[0] != r[j] && oj[1] != r[j]) bad = true;
        r[j + 1] = oj[0] == r[j] ? oj[1] : oj[0];
      }
      if (fn.closed && r[k] != r[0]) bad = true;
    }
    for (int j = 0; j < k; ++j) {
      const int64_t e = order[fn.first + j];
      const int64_t x = fn.first + j;
      // slot labelling (p, q, r_j, r_{j+1}) -> original local vertex indices
      int perm[4] = {-1, -1, -1, -1};
      const int32_t want[4] = {fn.p, fn.q, r[j], r[j + 1]};
      for (int s = 0; s < 4; ++s)
        for (int v = 0; v < 4; ++v)
          if (node(e, v) == want[s]) perm[s] = v;
      if (perm[0] < 0 || perm[1] < 0 || perm[2] < 0 || perm[3] < 0) {
        bad = true;
        continue;
      }
      int32_t sw[10];  // node word per slot
      for (int s = 0; s < 10; ++s) {
        const int a = s < 4 ? perm[s] : edge_slot(perm[ev[s - 4][0]], perm[ev[s - 4][1]]);
        const int32_t cw = word(e, a);
        sw[s] = cw;
      }
      bool interior = true;
      for (int s = 0; s < 10; ++s) interior = interior && ((static_cast<uint32_t>(sw[s]) >> 28) == 0u);
      const bool start = j == 0, end = j == k - 1;
      int32_t* w = wv.data() + kFanWords * size_t(x);
      for (int q = 0; q < kFanWords; ++q) w[q] = 0;
      w[0] = (start ? kFanStart : 0) | (end ? kFanEnd : 0) | (fn.closed ? kFanClosed : 0) | (interior ? kFanInterior : 0);
      // gathers: the rows this element adds
      if (start) {
        // p, q, m, r0, mid(p,r0), mid(q,r0), r1, mid(p,r1), mid(q,r1), mid(r0,r1)
        const int ss[10] = {0, 1, 4, 2, 6, 5, 3, 7, 8, 9};
        for (int q = 0; q < 10; ++q) w[1 + q] = sw[ss[q]];
      } else {
        if (!(end && fn.closed)) {
          w[1] = sw[3];
          w[2] = sw[7];
          w[3] = sw[8];
        } else {
          w[1] = w[2] = w[3] = -1;
        }
        w[4] = sw[9];
      }
      // coefficient record in slot order, volume from the original orientation
      double v[4][3], jm[3][3], inv[3][3];
      for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 3; ++c) v[a][c] = rnd(m.coords[3 * size_t(op.host_conn[e * 10 + perm[a]]) + c]);
      for (int c = 0; c < 3; ++c)
        for (int rr = 0; rr < 3; ++rr) jm[rr][c] = v[c + 1][rr] - v[0][rr];
      if (!inv3(jm, inv)) {
        bad = true;
        continue;
      }
      double rec[12];
      for (int kk = 0; kk < 3; ++kk)
        for (int d = 0; d < 3; ++d) rec[3 * kk + d] = inv[kk][d];
      rec[9] = coef64[12 * e + 9] / 20.0;
      rec[10] = coef64[12 * e + 10] / 20.0;
      rec[11] = 0.0;
      unsigned char* dst = cf.data() + size_t(x) * 12 * ts;
      for (int q = 0; q < 12; ++q) {
        if (fp32) {
          const float xx = static_cast<float>(rec[q]);
          std::memcpy(dst + q * 4, &xx, 4);
        } else {
          std::memcpy(dst + q * 8, &rec[q], 8);
        }
      }
    }
  }
  if (bad) validation("fan plan: inconsistent edge fan or degenerate element");
  setup_mark("fan: records");
  auto plan = std::make_unique<EbeFanPlan>();
  plan->n_units = U;
  plan->group_split = split;
  std::vector<int32_t> uf(size_t(U) + 1);
  int64_t closed_elems = 0;
  for (int32_t i = 0; i < U; ++i) {
    uf[i] = fans[i].first;
    if (fans[i].closed) closed_elems += fans[i].k;
  }
  uf[U] = static_cast<int32_t>(E);
  plan->closed_fraction = E ? double(closed_elems) / double(E) : 0.0;
  plan->mean_k = U ? double(E) / double(U) : 0.0;
  int64_t rows = 0;
  for (int32_t i = 0; i < U; ++i) rows += 4 * int64_t(fans[i].k) + (fans[i].closed ? 3 : 6);
  plan->rows_per_element = E ? double(rows) / double(E) : 0.0;
  plan->ufirst.upload(uf);
  plan->words.upload(wv);
  plan->coef.upload(cf);
  TS_CUDA(cudaDeviceSynchronize());  // the host staging arrays are released on return
  op.fan = std::move(plan);
}

}  // namespace tsg
