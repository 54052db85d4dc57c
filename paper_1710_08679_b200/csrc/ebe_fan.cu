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
#include <type_traits>
#include <vector>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {
namespace {

// step word record: 16 int32 = [flags, p, q, m, r0, mid(p,r0), mid(q,r0) (fan start only),
// M triple r_{j+1}, mid(p,.), mid(q,.) (-1: r_0), B triple r_{j+2} (-1: r_0 / no second element),
// ring edges e_j, e_{j+1} (-1: none), 0]; a row word is node | dof-mask bits << 28 (bare node ids
// in interior steps: the kInterior fast paths)
enum : int32_t { kFanStart = 1, kFanEnd = 2, kFanClosed = 4, kFanInterior = 8, kFanSingle = 16 };
constexpr int kFanWords = 16;
constexpr int kHdrSlots = 6;                    // p, q, m, r0, mid(p,r0), mid(q,r0)
constexpr int kRingBase = 2 * kHdrSlots;        // 5 ring-vertex triples
constexpr int kEdgeBase = kRingBase + 15;       // 4 ring edges
constexpr int kR0Base = kEdgeBase + 4;          // r0 partial sums of a closed fan
constexpr int kFanSlots = kR0Base + 3;          // row slots per lane group
constexpr int kRowV = 3;                        // lane vectors per row slot

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

// one lane's 3 components of a row slot
template <typename V>
__device__ __forceinline__ void load_row(const V* p, V (&r)[3]) {
  r[0] = p[0]; r[1] = p[1]; r[2] = p[2];
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
  constexpr int RCH = 24 / TPC;   // 16-byte chunks of a step's two coefficient records
  constexpr int RS = TPE * kRowV; // lane vectors per row slot
  extern __shared__ __align__(16) unsigned char smem[];
  const int grp = threadIdx.x / TPE;
  const int lane = threadIdx.x % TPE;
  V* const ug = reinterpret_cast<V*>(smem) + size_t(grp) * kFanSlots * RS + lane * kRowV;  // this lane's slot 0
  T* const cg = reinterpret_cast<T*>(smem + size_t(NT) * kFanSlots * kRowV * sizeof(V)) + size_t(grp) * 48;
  int4* const wg =
      reinterpret_cast<int4*>(smem + size_t(NT) * kFanSlots * kRowV * sizeof(V) + size_t(GROUPS) * 48 * sizeof(T)) +
      size_t(grp) * 12;
  const int col = lane * CPT;
  const T* const ub = u + col;
  T* const fb = f + col;
  const int32_t G = gridDim.x * GROUPS;

  // rows: interior steps carry bare node ids (no mask bits), so one IMAD addresses a row; the
  // interior / boundary choice is a compile-time flag (PL) of the step's whole gather or scatter
  // block, so neither path is predicated into the other
  auto gather = [&](auto PL, int32_t w, V* dst) {
    if constexpr (decltype(PL)::value) {
      const T* src = ub + static_cast<size_t>(static_cast<uint32_t>(w)) * (3 * B);
#pragma unroll
      for (int c = 0; c < 3; ++c) cpa(dst + c, src + c * B, int(sizeof(V)), sizeof(V));
    } else {
      const T* src = ub + static_cast<size_t>(static_cast<uint32_t>(w) & 0x0FFFFFFFu) * (3 * B);
      const unsigned mk = static_cast<unsigned>(w) >> 28;
#pragma unroll
      for (int c = 0; c < 3; ++c) cpa(dst + c, src + c * B, ((mk >> c) & 1u) ? 0 : int(sizeof(V)), sizeof(V));
    }
  };
  auto red = [&](auto PL, int32_t w, const V (&v)[3]) {
    if constexpr (decltype(PL)::value) {
      T* dst = fb + static_cast<size_t>(static_cast<uint32_t>(w)) * (3 * B);
#pragma unroll
      for (int c = 0; c < 3; ++c) red_lane(reinterpret_cast<V*>(dst + c * B), v[c]);
    } else {
      T* dst = fb + static_cast<size_t>(static_cast<uint32_t>(w) & 0x0FFFFFFFu) * (3 * B);
      const unsigned mk = static_cast<unsigned>(w) >> 28;
#pragma unroll
      for (int c = 0; c < 3; ++c) red_p(reinterpret_cast<V*>(dst + c * B), v[c], (mk >> c) & 1u);
    }
  };
  // three rows of partial sums
  auto red3 = [&](bool plain, const int32_t (&w)[3], const V (&v)[3][3]) {
    if (plain) {
      red(std::true_type{}, w[0], v[0]);
      red(std::true_type{}, w[1], v[1]);
      red(std::true_type{}, w[2], v[2]);
    } else {
      red(std::false_type{}, w[0], v[0]);
      red(std::false_type{}, w[1], v[1]);
      red(std::false_type{}, w[2], v[2]);
    }
  };
  auto red1 = [&](bool plain, int32_t w, const V (&v)[3]) {
    if (plain) red(std::true_type{}, w, v);
    else red(std::false_type{}, w, v);
  };
  auto fetch_words = [&](int32_t x, int ws) {
    if (x >= 0)
      for (int q = lane; q < 4; q += TPE) cpa(wg + 4 * ws + q, words + 4 * static_cast<size_t>(x) + q, 16, 16);
  };

  // slot allocation: ring triples rotate (5), ring edges rotate (4), fan headers alternate (2)
  struct Slots {
    int hdr, m, b, e0, e1;
  };
  int ring_next = 0, edge_next = 0, hdr_last = 1;
  auto ring_alloc = [&]() {
    const int r = ring_next;
    ring_next = ring_next == 4 ? 0 : ring_next + 1;
    return r;
  };
  auto edge_alloc = [&]() {
    const int r = edge_next;
    edge_next = (edge_next + 1) & 3;
    return r;
  };
  auto issue_rows = [&](auto PL, const int4& w0, const int4& w1, const int4& w2, const int4& w3, const Slots& st) {
    if (w0.x & kFanStart) {
      V* h = ug + st.hdr * (kHdrSlots * RS);
      gather(PL, w0.y, h);           // p
      gather(PL, w0.z, h + RS);      // q
      gather(PL, w0.w, h + 2 * RS);  // m
      gather(PL, w1.x, h + 3 * RS);  // r0
      gather(PL, w1.y, h + 4 * RS);  // mid(p, r0)
      gather(PL, w1.z, h + 5 * RS);  // mid(q, r0)
    }
    if (st.m >= 0) {  // M = r_{j+1} (else r0, in the header)
      V* r = ug + (kRingBase + 3 * st.m) * RS;
      gather(PL, w1.w, r);
      gather(PL, w2.x, r + RS);
      gather(PL, w2.y, r + 2 * RS);
    }
    if (st.b >= 0) {  // B = r_{j+2} (else r0, or no second element)
      V* r = ug + (kRingBase + 3 * st.b) * RS;
      gather(PL, w2.z, r);
      gather(PL, w2.w, r + RS);
      gather(PL, w3.x, r + 2 * RS);
    }
    gather(PL, w3.y, ug + (kEdgeBase + st.e0) * RS);
    if (w3.z != -1) gather(PL, w3.z, ug + (kEdgeBase + st.e1) * RS);
  };
  auto issue = [&](int32_t x, int ws, int rs) -> Slots {
    Slots st{hdr_last, -1, -1, 0, 0};
    if (x < 0) return st;
    const int4* w = wg + 4 * ws;
    const int4 w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3];
    const int32_t fl = w0.x;
    for (int q = lane; q < RCH; q += TPE) cpa(cg + 24 * rs + q * TPC, coef + 24 * static_cast<size_t>(x) + q * TPC, 16, 16);
    if (fl & kFanStart) {
      hdr_last ^= 1;
      st.hdr = hdr_last;
    }
    if (w1.w != -1) st.m = ring_alloc();
    if (w2.z != -1) st.b = ring_alloc();
    st.e0 = edge_alloc();
    if (w3.z != -1) st.e1 = edge_alloc();
    if (fl & kFanInterior) issue_rows(std::true_type{}, w0, w1, w2, w3, st);
    else issue_rows(std::false_type{}, w0, w1, w2, w3, st);
    return st;
  };

  // pipeline: step t (two elements of a fan) is computed while the rows of step t+1 stream in
  // and the words of step t+2 are fetched (word slots mod 3, record slots mod 2)
  FanCursor cur;
  cur.init(ufirst, u0 + static_cast<int32_t>(blockIdx.x) * GROUPS + grp, u1, G);
  int32_t xn = cur.x;
  cur.advance(ufirst, u1, G);
  fetch_words(xn, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  Slots stn = issue(xn, 0, 0);
  fetch_words(cur.x, 1);
  asm volatile("cp.async.commit_group;" ::: "memory");

  int wsc = 0, rsc = 0;
  int aslot = -1;                                      // ring triple of A (-1: r0 in the header)
  int32_t hw[6] = {0, 0, 0, 0, 0, 0}, aw[3] = {0, 0, 0};  // p q m r0 rows of the fan; A rows
  V S[3][3], FA[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) S[i][c] = FA[i][c] = O::zero();

  while (__any_sync(0xffffffffu, xn >= 0)) {
    const int32_t xc = xn;
    const Slots sc = stn;
    xn = cur.x;
    cur.advance(ufirst, u1, G);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const int wsn = wsc == 2 ? 0 : wsc + 1, ws2 = wsn == 2 ? 0 : wsn + 1;
    stn = issue(xn, wsn, rsc ^ 1);
    fetch_words(cur.x, ws2);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (xc >= 0) {
      const int4* w = wg + 4 * wsc;
      const int4 w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3];
      const int32_t fl = w0.x;
      const bool start = (fl & kFanStart) != 0, end = (fl & kFanEnd) != 0, closed = (fl & kFanClosed) != 0,
                 single = (fl & kFanSingle) != 0, plain = (fl & kFanInterior) != 0;
      if (start) {
        hw[0] = w0.y; hw[1] = w0.z; hw[2] = w0.w; hw[3] = w1.x; hw[4] = w1.y; hw[5] = w1.z;
        aw[0] = w1.x; aw[1] = w1.y; aw[2] = w1.z;
        aslot = -1;
      }
      const int32_t mw[3] = {w1.w != -1 ? w1.w : hw[3], w1.w != -1 ? w2.x : hw[4], w1.w != -1 ? w2.y : hw[5]};
      const V* h = ug + sc.hdr * (kHdrSlots * RS);
      const V* rm = sc.m < 0 ? h + 3 * RS : ug + (kRingBase + 3 * sc.m) * RS;
      V* const park = ug + kR0Base * RS;
      V sv[3][3];  // p, q, m rows (both elements)
      load_row(h, sv[0]);
      load_row(h + RS, sv[1]);
      load_row(h + 2 * RS, sv[2]);
      V mv[3][3];  // M rows: element j's B, element j+1's A (loaded once)
      load_row(rm, mv[0]);
      load_row(rm + RS, mv[1]);
      load_row(rm + 2 * RS, mv[2]);
      V FM[3][3];
      {  // element j = (p, q, r_j, r_{j+1}): A = r_j, B = M
        T rec[12];
        load_rec(cg + 24 * rsc, rec);
        V b[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) b[k][d] = O::splat(rec[3 * k + d]);
        const V lp = O::splat(rec[9]), mp = O::splat(rec[10]);
        const V* ra = aslot < 0 ? h + 3 * RS : ug + (kRingBase + 3 * aslot) * RS;
        V uu[10][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uu[0][c] = sv[0][c];
          uu[1][c] = sv[1][c];
          uu[4][c] = sv[2][c];
        }
        load_row(ra, uu[2]);
        load_row(ra + RS, uu[6]);
        load_row(ra + 2 * RS, uu[5]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uu[3][c] = mv[0][c];
          uu[7][c] = mv[1][c];
          uu[8][c] = mv[2][c];
        }
        load_row(ug + (kEdgeBase + sc.e0) * RS, uu[9]);
        V FE[3];
        tet10_product_acc<0x077u>(uu, b, lp, mp, [&](int s, int c) -> V& {
          return s == 0 ? S[0][c] : s == 1 ? S[1][c] : s == 4 ? S[2][c] : s == 2 ? FA[0][c] : s == 6 ? FA[1][c]
               : s == 5 ? FA[2][c] : s == 3 ? FM[0][c] : s == 7 ? FM[1][c] : s == 8 ? FM[2][c] : FE[c];
        });
        if (start && closed) {  // r_0 of a closed fan: parked until its last element
#pragma unroll
          for (int i = 0; i < 3; ++i) store_row(park + i * RS, FA[i]);
        } else {
          red3(plain, aw, FA);
        }
        red1(plain, w3.y, FE);
      }
      if (!single) {  // element j+1 = (p, q, r_{j+1}, r_{j+2}): A = M, B (into FA's registers)
        T rec[12];
        load_rec(cg + 24 * rsc + 12, rec);
        V b[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) b[k][d] = O::splat(rec[3 * k + d]);
        const V lp = O::splat(rec[9]), mp = O::splat(rec[10]);
        const V* rb = sc.b < 0 ? h + 3 * RS : ug + (kRingBase + 3 * sc.b) * RS;
        V uu[10][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uu[0][c] = sv[0][c];
          uu[1][c] = sv[1][c];
          uu[4][c] = sv[2][c];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uu[2][c] = mv[0][c];
          uu[6][c] = mv[1][c];
          uu[5][c] = mv[2][c];
        }
        load_row(rb, uu[3]);
        load_row(rb + RS, uu[7]);
        load_row(rb + 2 * RS, uu[8]);
        load_row(ug + (kEdgeBase + sc.e1) * RS, uu[9]);
        V FE[3];
        tet10_product_acc<0x077u>(uu, b, lp, mp, [&](int s, int c) -> V& {
          return s == 0 ? S[0][c] : s == 1 ? S[1][c] : s == 4 ? S[2][c] : s == 2 ? FM[0][c] : s == 6 ? FM[1][c]
               : s == 5 ? FM[2][c] : s == 3 ? FA[0][c] : s == 7 ? FA[1][c] : s == 8 ? FA[2][c] : FE[c];
        });
        red3(plain, mw, FM);
        red1(plain, w3.z, FE);
        // the step's last rows: B = r_{j+2} (r_0 of a closed fan: + its parked sums)
        const int32_t bw[3] = {w2.z != -1 ? w2.z : hw[3], w2.z != -1 ? w2.w : hw[4], w2.z != -1 ? w3.x : hw[5]};
        if (end) {
          if (closed)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              V r[3];
              load_row(park + i * RS, r);
#pragma unroll
              for (int c = 0; c < 3; ++c) FA[i][c] = O::add(FA[i][c], r[c]);
            }
          red3(plain, bw, FA);
        } else {
          aw[0] = bw[0]; aw[1] = bw[1]; aw[2] = bw[2];
          aslot = sc.b;
        }
      } else {  // a fan's odd last element: its B = M is the fan's last ring vertex (r_0 if closed)
        if (closed)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            V r[3];
            load_row(park + i * RS, r);
#pragma unroll
            for (int c = 0; c < 3; ++c) FM[i][c] = O::add(FM[i][c], r[c]);
          }
        red3(plain, mw, FM);
      }
      if (end) {  // p, q, m; the next fan starts from zero partial sums
        {
          const int32_t sw3[3] = {hw[0], hw[1], hw[2]};
          red3(plain, sw3, S);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int c = 0; c < 3; ++c) S[i][c] = FA[i][c] = O::zero();
        aslot = -1;
      }
    }
    __syncwarp();
    wsc = wsn;
    rsc ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <typename T, typename V, int B>
size_t fan_smem() {
  constexpr int CPT = LaneOps<V>::kCols, TPE = (B + CPT - 1) / CPT, NT = 128, GROUPS = NT / TPE;
  return size_t(NT) * kFanSlots * kRowV * sizeof(V) + size_t(GROUPS) * 48 * sizeof(T) + size_t(GROUPS) * 12 * 16;
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
    const int64_t step = strided_launch_units(int64_t(grid) * GROUPS, int64_t(q1) - q0);
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

  // steps: each fan's elements two by two (an odd fan ends with a single-element step)
  std::vector<int32_t> sfirst(size_t(U) + 1, 0);
  for (int32_t i = 0; i < U; ++i) sfirst[i + 1] = sfirst[i] + (fans[i].k + 1) / 2;
  const int64_t NS = sfirst[U];
  const size_t ts = fp32 ? 4 : 8;
  HostVec<int32_t> wv(size_t(NS) * kFanWords);
  HostVec<unsigned char> cf(size_t(NS) * 24 * ts);
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
    // per element: slot words (p, q, r_j, r_{j+1} labelling) and the coefficient record
    std::vector<std::array<int32_t, 10>> sw(k);
    std::vector<std::array<double, 12>> rec(k);
    bool interior_all = true;
    for (int j = 0; j < k && !bad; ++j) {
      const int64_t e = order[fn.first + j];
      int perm[4] = {-1, -1, -1, -1};
      const int32_t want[4] = {fn.p, fn.q, r[j], r[j + 1]};
      for (int q = 0; q < 4; ++q)
        for (int v = 0; v < 4; ++v)
          if (node(e, v) == want[q]) perm[q] = v;
      if (perm[0] < 0 || perm[1] < 0 || perm[2] < 0 || perm[3] < 0) {
        bad = true;
        break;
      }
      for (int q = 0; q < 10; ++q) {
        const int a = q < 4 ? perm[q] : edge_slot(perm[ev[q - 4][0]], perm[ev[q - 4][1]]);
        sw[j][q] = word(e, a);
      }
      double v[4][3], jm[3][3], inv[3][3];
      for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 3; ++c) v[a][c] = rnd(m.coords[3 * size_t(op.host_conn[e * 10 + perm[a]]) + c]);
      for (int c = 0; c < 3; ++c)
        for (int rr = 0; rr < 3; ++rr) jm[rr][c] = v[c + 1][rr] - v[0][rr];
      if (!inv3(jm, inv)) {
        bad = true;
        break;
      }
      for (int kk = 0; kk < 3; ++kk)
        for (int d = 0; d < 3; ++d) rec[j][3 * kk + d] = inv[kk][d];
      rec[j][9] = coef64[12 * e + 9] / 20.0;  // lambda V / 20, mu V / 20: original orientation
      rec[j][10] = coef64[12 * e + 10] / 20.0;
      rec[j][11] = 0.0;
      // consecutive elements share p, q, m and the ring vertex between them
      if (j > 0) {
        const int sa[3] = {0, 1, 4};
        for (int q : sa) bad = bad || sw[j][q] != sw[j - 1][q];
        bad = bad || sw[j][2] != sw[j - 1][3] || sw[j][6] != sw[j - 1][7] || sw[j][5] != sw[j - 1][8];
      }
    }
    if (bad) continue;
    const int nsteps = (k + 1) / 2;
    for (int st = 0; st < nsteps; ++st) {
      const int j = 2 * st;
      const bool single = j + 1 == k, start = st == 0, end = st == nsteps - 1;
      bool interior = true;
      for (int q = 0; q < 10; ++q) interior = interior && ((static_cast<uint32_t>(sw[j][q]) >> 28) == 0u);
      if (!single)
        for (int q = 0; q < 10; ++q) interior = interior && ((static_cast<uint32_t>(sw[j + 1][q]) >> 28) == 0u);
      interior_all = interior_all && interior;
      int32_t* w = wv.data() + kFanWords * size_t(sfirst[fi] + st);
      for (int q = 0; q < kFanWords; ++q) w[q] = -1;
      w[0] = (start ? kFanStart : 0) | (end ? kFanEnd : 0) | (fn.closed ? kFanClosed : 0) |
             (interior ? kFanInterior : 0) | (single ? kFanSingle : 0);
      w[15] = 0;
      if (start) {  // p, q, m, r0, mid(p,r0), mid(q,r0)
        w[1] = sw[0][0]; w[2] = sw[0][1]; w[3] = sw[0][4]; w[4] = sw[0][2]; w[5] = sw[0][6]; w[6] = sw[0][5];
      }
      if (!(fn.closed && j + 1 == k)) {  // M = r_{j+1}
        w[7] = sw[j][3]; w[8] = sw[j][7]; w[9] = sw[j][8];
      }
      if (!single && !(fn.closed && j + 2 == k)) {  // B = r_{j+2}
        w[10] = sw[j + 1][3]; w[11] = sw[j + 1][7]; w[12] = sw[j + 1][8];
      }
      w[13] = sw[j][9];
      if (!single) w[14] = sw[j + 1][9];
      unsigned char* dst = cf.data() + size_t(sfirst[fi] + st) * 24 * ts;
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 12; ++q) {
          const double x = (h == 1 && single) ? 0.0 : rec[j + h][q];
          if (fp32) {
            const float xx = static_cast<float>(x);
            std::memcpy(dst + (12 * h + q) * 4, &xx, 4);
          } else {
            std::memcpy(dst + (12 * h + q) * 8, &x, 8);
          }
        }
    }
    (void)interior_all;
  }
  if (bad) validation("fan plan: inconsistent edge fan or degenerate element");
  setup_mark("fan: records");
  auto plan = std::make_unique<EbeFanPlan>();
  plan->n_units = U;
  plan->group_split = split;
  std::vector<int32_t> uf(sfirst.begin(), sfirst.end());
  int64_t closed_elems = 0;
  for (int32_t i = 0; i < U; ++i)
    if (fans[i].closed) closed_elems += fans[i].k;
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
