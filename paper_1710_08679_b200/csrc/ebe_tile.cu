// ebe_tile.cu — chunk-aggregated EBE sweep (the production sm_100a kernel).
//
// Replaces EbeOperator<T>::apply's element loop (ebe_operator.hpp:112-188):
// f += sum_e Q_e K_e Q_e^T u, with the reference's masking (gather zeroes
// constrained inputs, scatter skips constrained outputs, :154-155, :182).
//
// Why this shape (measured on B200, scripts/micro/gather_scatter.cu,
// profiles/r01_ebe_memory_paths.txt): a per-element vector-RED scatter of the
// 30 x r outputs costs ~1.0 ms for the 10M-DOF box at r = 16 on its own — the
// L2 atomic units, not DRAM, are the limit — while the lean element product is
// FP32-pipe bound at ~0.54 ms (FFMA2 issues at 0.5 / clk / SMSP). So the sweep
// aggregates in shared memory first:
//
//   * elements are cut into chunks of kChunk consecutive (Morton-ordered)
//     elements; per chunk the setup records its distinct nodes, each element's
//     local node slots, and each node's incidence list (chunk "record");
//   * TILE:    the chunk's node rows u[node][3][r] are copied once into shared
//              memory with coalesced 16-byte cp.async (constrained dofs are
//              zero-filled by the copy engine: src-size 0);
//   * COMPUTE: a lane group per element (TPE threads x CPT cases) runs the
//              exact lean tet10/tet4 product (element_kernels.cuh) from the
//              tile and parks its 3*NPE x r outputs in a per-element slot of a
//              bank-padded contribution buffer (plain stores, no atomics);
//   * REDUCE:  threads own 16-byte pieces of the chunk's node rows, sum the
//              node's incidences from shared memory and issue one vector RED
//              per piece — ~3 node rows per element reach L2 instead of 10,
//              in full 32-byte sectors. Constrained dofs are skipped (f holds
//              the masked identity, written before the sweep).
//
// The chunk records, the tile and the coefficients of chunk k+1 stream in
// (cp.async) while chunk k reduces; records are prefetched two chunks ahead.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "ebe.h"
#include "element_kernels.cuh"

namespace tsg {

namespace {

constexpr int kChunkDefault = 32;  // elements per chunk (one lane group each)
constexpr int kChunkTet4 = 32;  // 64 and 128 measured slower (profiles/r01_ebe_tile.txt)

__device__ __forceinline__ void cpa16(void* s, const void* g, int src) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
}
__device__ __forceinline__ void cpa8(void* s, const void* g, int src) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
}
__device__ __forceinline__ void cpa4(void* s, const void* g, int src) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(a), "l"(g), "r"(src) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cpa(void* s, const void* g, int src) {
  if constexpr (BYTES == 16) cpa16(s, g, src);
  else if constexpr (BYTES == 8) cpa8(s, g, src);
  else cpa4(s, g, src);
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---- reduction units: UW scalars of T (16, 8 or 4 bytes) ----------------------
template <typename T, int UW> struct Unit;
template <> struct Unit<float, 4> {
  using type = float4;
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static float4 add(float4 a, float4 b) {
    const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
    const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  }
  __device__ static void red(float* p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
  }
};
template <> struct Unit<float, 2> {
  using type = float2;
  __device__ static float2 zero() { return make_float2(0.f, 0.f); }
  __device__ static float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
  __device__ static void red(float* p, float2 v) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
  }
};
template <> struct Unit<float, 1> {
  using type = float;
  __device__ static float zero() { return 0.f; }
  __device__ static float add(float a, float b) { return a + b; }
  __device__ static void red(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
  }
};
template <> struct Unit<double, 2> {
  using type = double2;
  __device__ static double2 zero() { return make_double2(0.0, 0.0); }
  __device__ static double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  __device__ static void red(double* p, double2 v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v.x) : "memory");
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + 1), "d"(v.y) : "memory");
  }
};
template <> struct Unit<double, 1> {
  using type = double;
  __device__ static double zero() { return 0.0; }
  __device__ static double add(double a, double b) { return a + b; }
  __device__ static void red(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  }
};

// Compile-time geometry of one kernel instance.
template <typename T, typename V, int NPE, int B, int kChunk>
struct TileCfg {
  static constexpr int CPT = LaneOps<V>::kCols;       // cases per thread
  static constexpr int TPE = (B + CPT - 1) / CPT;     // threads per element
  static constexpr int NT = kChunk * TPE;             // threads per block
  static constexpr int ROW = 3 * B;                   // T per node row [3][B]
  static constexpr int SEG = B * int(sizeof(T));      // bytes of one dof row
  static constexpr int UB = SEG % 16 == 0 ? 16 : (SEG % 8 == 0 ? 8 : 4);  // copy / reduce unit bytes
  static constexpr int UW = UB / int(sizeof(T));      // T per unit
  static constexpr int UPD = B / UW;                  // units per dof row
  static constexpr int UPN = 3 * UPD;                 // units per node row
  // element slot stride: pad so consecutive elements' dof rows start in
  // different bank groups (stride = SEG mod 128 bytes)
  static constexpr int RAW = NPE * 3 * SEG;
  static constexpr int PADB = SEG >= 128 ? 0 : ((SEG - RAW % 128) % 128 + 128) % 128;
  static constexpr int ES = (RAW + PADB) / int(sizeof(T));  // T per element slot
};

struct RecHdr {
  int32_t n_nodes, n_elems, e_begin, n16;
};

// Layout of a chunk record (16-byte aligned sections), see build_tile_plan.
struct RecView {
  const RecHdr* hdr;
  const uint32_t* nodes;   // [L] node | dof-mask bits << 28
  const uint16_t* inc_off; // [L+1]
  const uint16_t* inc;     // [ne*NPE] (slot << 4) | local node a, grouped by node
  const uint16_t* lconn;   // [ne*NPE] tile row of (element, a)
};
__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }
template <int NPE>
__device__ __forceinline__ RecView rec_view(const unsigned char* base) {
  RecView v;
  v.hdr = reinterpret_cast<const RecHdr*>(base);
  const int L = v.hdr->n_nodes, ne = v.hdr->n_elems;
  int off = 16;
  v.nodes = reinterpret_cast<const uint32_t*>(base + off);
  off += align16(4 * L);
  v.inc_off = reinterpret_cast<const uint16_t*>(base + off);
  off += align16(2 * (L + 1));
  v.inc = reinterpret_cast<const uint16_t*>(base + off);
  off += align16(2 * ne * NPE);
  v.lconn = reinterpret_cast<const uint16_t*>(base + off);
  return v;
}

template <typename T, typename V, int NPE, int B, int kChunk, bool ROWRED>
__global__ void __launch_bounds__(TileCfg<T, V, NPE, B, kChunk>::NT)
k_ebe_tile(const uint4* __restrict__ rec, const uint32_t* __restrict__ rec_off, int32_t c_begin, int32_t n_chunks,
           int rec_max, int lmax, const T* __restrict__ coef, const T* __restrict__ u, T* __restrict__ f) {
  using Cfg = TileCfg<T, V, NPE, B, kChunk>;
  using O = LaneOps<V>;
  using U = Unit<T, Cfg::UW>;
  using UV = typename U::type;
  constexpr int NT = Cfg::NT, TPE = Cfg::TPE, CPT = Cfg::CPT, ROW = Cfg::ROW, ES = Cfg::ES;
  constexpr int UB = Cfg::UB, UW = Cfg::UW, UPD = Cfg::UPD, UPN = Cfg::UPN;
  constexpr int CB = kChunk * 12 * int(sizeof(T));  // coefficient bytes per chunk
  extern __shared__ __align__(16) unsigned char smem[];
  T* contrib = reinterpret_cast<T*>(smem);                                   // [kChunk][ES]
  T* tile = contrib + kChunk * ES;                                           // [lmax][ROW]
  T* cf = tile + static_cast<size_t>(lmax) * ROW;                            // [kChunk][12]
  int* incoff = reinterpret_cast<int*>(cf + kChunk * 12);                   // [kChunk * NPE]
  unsigned char* meta = reinterpret_cast<unsigned char*>(incoff + kChunk * NPE);  // [3][rec_max]

  const int tid = threadIdx.x;
  const int G = gridDim.x;

  auto load_rec = [&](int c, int stage) {
    const uint32_t o = __ldg(rec_off + c), n = __ldg(rec_off + c + 1) - o;
    unsigned char* dst = meta + stage * rec_max;
    for (uint32_t i = tid; i < n; i += NT) cpa16(dst + 16 * i, rec + o + i, 16);
  };
  // Unit-loop mapping: thread tid < SN*UPN owns unit column j = tid % UPN of
  // every SN-th chunk node (fixed component / offset, no per-item division).
  constexpr int SN = NT / UPN;
  const bool uact = tid < SN * UPN;
  const int uj = tid % UPN, un0 = tid / UPN;
  const int uk = uj / UPD, ujj = (uj - uk * UPD) * UW;  // component, offset within the dof row
  const T* usrc = u + uj * UW;

  auto issue_tile = [&](int stage) {
    const RecView rv = rec_view<NPE>(meta + stage * rec_max);
    const int L = rv.hdr->n_nodes, ne = rv.hdr->n_elems, e0 = rv.hdr->e_begin;
    if (uact) {
      T* dst = tile + un0 * ROW + uj * UW;
#pragma unroll 2
      for (int n = un0; n < L; n += SN, dst += SN * ROW) {
        const uint32_t w = rv.nodes[n];
        const bool live = !((w >> (28 + uk)) & 1u);
        cpa<UB>(dst, usrc + static_cast<size_t>(w & 0x0FFFFFFFu) * ROW, live ? UB : 0);
      }
    }
    const unsigned char* cs = reinterpret_cast<const unsigned char*>(coef + static_cast<size_t>(e0) * 12);
    for (int it = tid; it * 16 < ne * 12 * int(sizeof(T)); it += NT)
      cpa16(reinterpret_cast<unsigned char*>(cf) + 16 * it, cs + 16 * it, 16);
    (void)CB;
  };

  int c = c_begin + blockIdx.x;
  if (c >= n_chunks) return;
  load_rec(c, 0);
  cpa_commit();
  cpa_wait_all();
  __syncthreads();
  if (c + G < n_chunks) load_rec(c + G, 1);
  issue_tile(0);
  cpa_commit();
  int ms = 0;
  for (; c < n_chunks; c += G) {
    cpa_wait_all();
    __syncthreads();  // tile(c), coefficients(c), record(c+G) resident
    const unsigned char* mb = meta + ms * rec_max;
    const RecView rv = rec_view<NPE>(mb);
    const int L = rv.hdr->n_nodes, ne = rv.hdr->n_elems;
    // ---- COMPUTE: lane group g = element g of the chunk
    {
      const int g = tid / TPE, l = tid - (tid / TPE) * TPE;
      if (g < ne) {
        const T* cfe = cf + g * 12;
        V b[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) b[k][d] = O::splat(cfe[3 * k + d]);
        const V lp = O::splat(cfe[9]), mp = O::splat(cfe[10]);
        V uu[NPE][3];
        const uint16_t* lc = rv.lconn + g * NPE;
#pragma unroll
        for (int a = 0; a < NPE; ++a) {
          const T* row = tile + static_cast<int>(lc[a]) * ROW + l * CPT;
#pragma unroll
          for (int k = 0; k < 3; ++k) uu[a][k] = *reinterpret_cast<const V*>(row + k * B);
        }
        V ff[NPE][3];
        if constexpr (NPE == 10) tet10_product<V>(uu, b, lp, mp, ff);
        else tet4_product<V>(uu, b, lp, mp, ff);
        T* dst = contrib + g * ES + l * CPT;
#pragma unroll
        for (int a = 0; a < NPE; ++a)
#pragma unroll
          for (int k = 0; k < 3; ++k) *reinterpret_cast<V*>(dst + (a * 3 + k) * B) = ff[a][k];
      }
    }
    // incidence (slot << 4 | a) -> contribution row offset of this instance
    for (int i = tid; i < ne * NPE; i += NT) {
      const int sl = rv.inc[i];
      incoff[i] = (sl >> 4) * ES + (sl & 15) * 3 * B;
    }
    __syncthreads();  // contributions parked; tile and coefficient buffers free
    if (c + G < n_chunks) issue_tile((ms + 1) % 3);
    if (c + 2 * G < n_chunks) load_rec(c + 2 * G, (ms + 2) % 3);
    cpa_commit();
    // ---- REDUCE
    if constexpr (ROWRED) {
      // thread owns dof row k of every SR-th chunk node: one incidence walk per row
      constexpr int SR = NT / 3;
      if (tid < 3 * SR) {
        const int k = tid % 3;
        const T* cbase = contrib + k * B;
        for (int n = tid / 3; n < L; n += SR) {
          const uint32_t w = rv.nodes[n];
          if ((w >> (28 + k)) & 1u) continue;
          const int p1 = rv.inc_off[n + 1];
          int p = rv.inc_off[n];
          UV acc[UPD];
#pragma unroll
          for (int q = 0; q < UPD; ++q) acc[q] = *reinterpret_cast<const UV*>(cbase + incoff[p] + q * UW);
#pragma unroll 1
          for (++p; p < p1; ++p) {
            const T* src = cbase + incoff[p];
#pragma unroll
            for (int q = 0; q < UPD; ++q) acc[q] = U::add(acc[q], *reinterpret_cast<const UV*>(src + q * UW));
          }
          T* dst = f + static_cast<size_t>(w & 0x0FFFFFFFu) * ROW + k * B;
#pragma unroll
          for (int q = 0; q < UPD; ++q) U::red(dst + q * UW, acc[q]);
        }
      }
    } else if (uact) {
      // thread owns unit (uk, ujj) of every SN-th chunk node row
      const T* cbase = contrib + uk * B + ujj;
      const int* io = incoff;
      for (int n = un0; n < L; n += SN) {
        const uint32_t w = rv.nodes[n];
        if ((w >> (28 + uk)) & 1u) continue;  // constrained dof: identity row already in f
        const int p1 = rv.inc_off[n + 1];
        int p = rv.inc_off[n];
        UV acc = *reinterpret_cast<const UV*>(cbase + io[p]);
#pragma unroll 1
        for (++p; p < p1; ++p) acc = U::add(acc, *reinterpret_cast<const UV*>(cbase + io[p]));
        U::red(f + static_cast<size_t>(w & 0x0FFFFFFFu) * ROW + uk * B + ujj, acc);
      }
    }
    ms = (ms + 1) % 3;
  }
}


template <typename T, typename V, int NPE, int B, int kChunk, bool ROWRED>
bool launch_tile_c(const ts_ebe& op, const EbeTilePlan& plan, const T* u, T* f, cudaStream_t s, int32_t c0,
                   int32_t c1) {
  using Cfg = TileCfg<T, V, NPE, B, kChunk>;
  const size_t smem = sizeof(T) * (size_t(kChunk) * Cfg::ES + size_t(plan.lmax) * Cfg::ROW + kChunk * 12) +
                      sizeof(int) * kChunk * NPE + 3 * size_t(plan.rec_max);
  if (smem > 227 * 1024) return false;
  auto kern = k_ebe_tile<T, V, NPE, B, kChunk, ROWRED>;
  const KernelFit fit = kernel_fit<k_ebe_tile<T, V, NPE, B, kChunk, ROWRED>>(Cfg::NT, smem);
  const int sms = fit.sms, per_sm = fit.per_sm;
  if (per_sm < 1) return false;
  if (c1 <= c0) return true;
  const int grid = std::max(1, std::min(c1 - c0, sms * per_sm));
  kern<<<grid, Cfg::NT, smem, s>>>(reinterpret_cast<const uint4*>(plan.rec.get()), plan.rec_off.get(), c0,
                                   c1, plan.rec_max, plan.lmax, reinterpret_cast<const T*>(op.coef.get()),
                                   u, f);
  TS_CUDA_LAUNCH();
  return true;
}

template <typename T, typename V, int NPE, int B>
bool launch_tile_b(const ts_ebe& op, const EbeTilePlan& plan, const T* u, T* f, cudaStream_t s, int32_t c0,
                   int32_t c1) {
  constexpr int TPE = TileCfg<T, V, NPE, B, 1>::TPE;
  switch (plan.chunk) {
    case 16: return launch_tile_c<T, V, NPE, B, 16, false>(op, plan, u, f, s, c0, c1);
    case 32: return launch_tile_c<T, V, NPE, B, 32, false>(op, plan, u, f, s, c0, c1);
    case 64:
      if constexpr (64 * TPE <= 1024) return launch_tile_c<T, V, NPE, B, 64, false>(op, plan, u, f, s, c0, c1);
      return false;
    case 128:
      if constexpr (128 * TPE <= 1024) return launch_tile_c<T, V, NPE, B, 128, false>(op, plan, u, f, s, c0, c1);
      return false;
    default: return false;
  }
}

template <typename T, typename V, int NPE>
bool launch_tile_npe(const ts_ebe& op, const T* u, T* f, int32_t batch, cudaStream_t s, int32_t c0, int32_t c1) {
  const EbeTilePlan& plan = *op.tile;
  switch (batch) {
    case 1: return launch_tile_b<T, T, NPE, 1>(op, plan, u, f, s, c0, c1);
    case 2: return launch_tile_b<T, V, NPE, 2>(op, plan, u, f, s, c0, c1);
    case 4: return launch_tile_b<T, V, NPE, 4>(op, plan, u, f, s, c0, c1);
    case 8: return launch_tile_b<T, V, NPE, 8>(op, plan, u, f, s, c0, c1);
    case 16: return launch_tile_b<T, V, NPE, 16>(op, plan, u, f, s, c0, c1);
    case 32:
      if constexpr (sizeof(T) == 4) return launch_tile_b<T, V, NPE, 32>(op, plan, u, f, s, c0, c1);
      return false;
    default: return false;
  }
}

}  // namespace

bool ebe_tile_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part) {
  if (!op.tile || op.tile->n_chunks == 0) return false;
  const int32_t c0 = part == 1 ? op.tile->group_chunk_split : 0;
  const int32_t c1 = part == 0 ? op.tile->group_chunk_split : op.tile->n_chunks;
  if (op.prec == 32) {
    const float* uu = static_cast<const float*>(u);
    float* ff = static_cast<float*>(f);
    return op.order == 2 ? launch_tile_npe<float, float2, 10>(op, uu, ff, batch, s, c0, c1)
                         : launch_tile_npe<float, float2, 4>(op, uu, ff, batch, s, c0, c1);
  }
  const double* uu = static_cast<const double*>(u);
  double* ff = static_cast<double*>(f);
  return op.order == 2 ? launch_tile_npe<double, double, 10>(op, uu, ff, batch, s, c0, c1)
                       : launch_tile_npe<double, double, 4>(op, uu, ff, batch, s, c0, c1);
}

// Chunk records from the Morton-ordered connectivity words (node | mask << 28).
void build_tile_plan(ts_ebe& op, const HostVec<int32_t>& conn_words, int conn_stride) {
  const int npe = op.npe;
  const int64_t E = op.n_elems;
  auto plan = std::make_unique<EbeTilePlan>();
  // elements per chunk: tet10 32 (one 256-thread block at r = 16); the light tet4
  // product amortises the per-chunk pipeline over more elements
  int kChunk = npe == 4 ? kChunkTet4 : kChunkDefault;
  if (const char* e = std::getenv(npe == 4 ? "TSGPU_TILE_CHUNK4" : "TSGPU_TILE_CHUNK")) {
    const int c = std::atoi(e);
    kChunk = (c == 16 || c == 32 || c == 64 || c == 128) ? c : kChunk;
  }
  plan->chunk = kChunk;
  // chunks never straddle the element-group boundary (boundary / interior sweeps)
  std::vector<int64_t> cstart;
  for (int64_t e = 0; e < op.group_split; e += kChunk) cstart.push_back(e);
  plan->group_chunk_split = static_cast<int32_t>(cstart.size());
  for (int64_t e = op.group_split; e < E; e += kChunk) cstart.push_back(e);
  plan->n_chunks = static_cast<int32_t>(cstart.size());
  const int32_t nc = plan->n_chunks;
  std::vector<std::vector<uint32_t>> recs(nc);
  std::vector<int> lmax_t(nc, 0);
#pragma omp parallel for schedule(static)
  for (int32_t c = 0; c < nc; ++c) {
    const int64_t e0 = cstart[c];
    const int64_t gend = e0 < op.group_split ? op.group_split : E;
    const int ne = static_cast<int>(std::min<int64_t>(kChunk, gend - e0));
    // distinct nodes in ascending id order (adjacent ids -> adjacent rows in HBM)
    std::vector<uint32_t> nodes(ne * npe);
    std::vector<uint16_t> lconn(ne * npe);
    for (int q = 0; q < ne * npe; ++q)
      nodes[q] = static_cast<uint32_t>(conn_words[(e0 + q / npe) * conn_stride + q % npe]);
    std::sort(nodes.begin(), nodes.end(),
              [](uint32_t x, uint32_t y) { return (x & 0x0FFFFFFFu) < (y & 0x0FFFFFFFu); });
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    for (int q = 0; q < ne * npe; ++q) {
      const uint32_t w = static_cast<uint32_t>(conn_words[(e0 + q / npe) * conn_stride + q % npe]);
      const auto it = std::lower_bound(nodes.begin(), nodes.end(), w,
                                       [](uint32_t x, uint32_t y) { return (x & 0x0FFFFFFFu) < (y & 0x0FFFFFFFu); });
      lconn[q] = static_cast<uint16_t>(it - nodes.begin());
    }
    const int L = static_cast<int>(nodes.size());
    std::vector<uint16_t> inc_off(L + 1, 0), inc(ne * npe);
    for (int q = 0; q < ne * npe; ++q) ++inc_off[lconn[q] + 1];
    for (int n = 0; n < L; ++n) inc_off[n + 1] += inc_off[n];
    std::vector<uint16_t> cur(inc_off.begin(), inc_off.end() - 1);
    for (int g = 0; g < ne; ++g)
      for (int a = 0; a < npe; ++a) inc[cur[lconn[g * npe + a]]++] = static_cast<uint16_t>((g << 4) | a);
    const int bytes = 16 + align16(4 * L) + align16(2 * (L + 1)) + 2 * align16(2 * ne * npe);
    std::vector<uint32_t> r(bytes / 4, 0);
    unsigned char* b = reinterpret_cast<unsigned char*>(r.data());
    const RecHdr h{L, ne, static_cast<int32_t>(e0), bytes / 16};
    std::memcpy(b, &h, sizeof h);
    int off = 16;
    std::memcpy(b + off, nodes.data(), 4 * L);
    off += align16(4 * L);
    std::memcpy(b + off, inc_off.data(), 2 * (L + 1));
    off += align16(2 * (L + 1));
    std::memcpy(b + off, inc.data(), 2 * ne * npe);
    off += align16(2 * ne * npe);
    std::memcpy(b + off, lconn.data(), 2 * ne * npe);
    recs[c].swap(r);
    lmax_t[c] = L;
  }
  std::vector<uint32_t> off(nc + 1, 0);
  int rec_max = 0, lmax = 0;
  int64_t tot_nodes = 0;
  for (int32_t c = 0; c < nc; ++c) {
    off[c + 1] = off[c] + static_cast<uint32_t>(recs[c].size() / 4);
    rec_max = std::max(rec_max, static_cast<int>(recs[c].size() * 4));
    lmax = std::max(lmax, lmax_t[c]);
    tot_nodes += lmax_t[c];
  }
  std::vector<uint32_t> all(static_cast<size_t>(off[nc]) * 4);
#pragma omp parallel for schedule(static)
  for (int32_t c = 0; c < nc; ++c) std::memcpy(all.data() + size_t(off[c]) * 4, recs[c].data(), recs[c].size() * 4);
  plan->rec_max = rec_max;
  plan->lmax = (lmax + 3) & ~3;  // keeps the coefficient buffer after the tile 16-byte aligned
  plan->nodes_per_elem = E ? double(tot_nodes) / double(E) : 0.0;
  plan->rec.upload(reinterpret_cast<const unsigned char*>(all.data()), all.size() * 4);
  plan->rec_off.upload(off);
  op.tile = std::move(plan);
}

}  // namespace tsg
