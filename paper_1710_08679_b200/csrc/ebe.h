// ebe.h — device-resident matrix-free EBE operator (EbeOperator<T>,
// ebe_operator.hpp:29-226), shared by the solver translation units.
#pragma once
#include <algorithm>
#include <array>
#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "ts_common.h"

// Greedy first-fit element coloring over shared nodes (build_coloring,
// ebe_operator.hpp:190-214), on sweep positions: no two elements of a color
// share a node, so a color's contributions land with plain read-add-writes and
// every node sums its elements in color order, independent of the batch width,
// the launch geometry and the run (ebe_color.cu).
struct EbeColorPlan {
  int n_colors = 0;
  std::vector<int32_t> color_ptr;  // [n_colors + 1] into elems
  tsg::DevBuf<int32_t> elems;      // sweep positions, color-major, ascending within a color
};

// Face-sharing element pairs for the pair sweep (ebe_pair.cu).
struct EbePairPlan {
  int32_t n_units = 0;           // pairs and singles in element order, per element group
  int32_t group_split = 0;       // units [0, split) cover element group 0
  double paired_fraction = 0.0;  // elements that are in a pair
  tsg::DevBuf<int32_t> conn;     // [units][16 | 8]: A's slots, B's own slots (3*node), mask words
  tsg::DevBuf<unsigned char> coef;  // [units][24] of T: A and B coefficient records
  tsg::DevBuf<int32_t> sched;       // unit-chunk counters of the dynamic schedule, one per launch slot
  mutable std::atomic<uint32_t> next_slot{0};  // launches take counter slots round-robin
};

// Edge fans for the fan sweep (ebe_fan.cu): element j of a fan around edge (p, q) is
// (p, q, r_j, r_{j+1}); elements are stored in fan order.
struct EbeFanPlan {
  int32_t n_units = 0;            // fans, in element-group order
  int32_t group_split = 0;        // fans [0, split) cover element group 0
  double closed_fraction = 0.0;   // elements in closed fans
  double mean_k = 0.0;            // elements per fan
  double rows_per_element = 0.0;  // node rows gathered (= reduced) per element
  tsg::DevBuf<int32_t> words;     // [steps][16]: flags, the rows a step (two elements) adds (node | mask << 28)
  tsg::DevBuf<unsigned char> coef;  // [steps][24] of T: the step's two slot-order coefficient records
  tsg::DevBuf<int32_t> ufirst;    // [U + 1] first step of each fan
};

// Elements sweep in slabs of their lowest vertex id (then Morton order), ebe.cu;
// TSGPU_EBE_SLABS overrides (1 = plain Morton)
constexpr int kEbeSlabs = 16;
int ebe_slab_count();
// Slab of an element whose lowest vertex id is v (of V vertices), S slabs. The first
// and last slabs are half as thick as the others: they are the host-buffer
// apply's pipeline fill (first upload) and drain (last download), ebe_stream.cu.
inline int ebe_slab_of(int64_t v, int64_t V, int S) {
  if (S <= 2) return static_cast<int>(std::min<int64_t>(S - 1, v * S / std::max<int64_t>(1, V)));
  constexpr int64_t kMid = 2;             // width of a middle slab in end-slab units
  const int64_t units = kMid * (S - 2) + 2;
  const int64_t k = v * units / std::max<int64_t>(1, V);
  if (k == 0) return 0;
  if (k >= units - 1) return S - 1;
  return static_cast<int>(1 + (k - 1) / kMid);
}

// Host-buffer streaming schedule (ebe_stream.cu): the pair units cut into
// chunks; node rows go up before the first chunk that reads them and come back
// after the last chunk that writes them.
struct EbeStreamPlan {
  bool usable = false;
  int chunks = 0;
  std::vector<int32_t> unit_ptr;                 // [chunks + 1] pair-unit ranges
  std::vector<int32_t> in_ptr, out_ptr;          // [chunks + 1] into in_runs / out_runs
  std::vector<std::array<int32_t, 2>> in_runs;   // node ranges [a, b) uploaded before chunk k
  std::vector<std::array<int32_t, 2>> out_runs;  // node ranges final after chunk k
  std::vector<int32_t> mdof_ptr;                 // [chunks + 1] into mdofs
  tsg::DevBuf<int32_t> mdofs;                    // constrained dofs by upload chunk
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done;
  cudaEvent_t ev_entry = nullptr;  // recorded on the legacy stream at entry: the pipeline waits on it
  ~EbeStreamPlan();
};

struct ts_ebe {
  int order = 2;   // 1 = tet4 on the vertex grid, 2 = tet10
  int npe = 10;
  int prec = 32;   // 32 | 64 : the reference's T
  int32_t n_nodes = 0;
  int32_t n_elems = 0;
  int32_t n_vertices = 0;  // mesh vertex count (the slab key's range)
  int n_slabs = kEbeSlabs; // element-order slabs (ebe_stream.cu chunks on them)
  bool has_mask = false;
  int conn_stride = 12;                 // int32 per element (npe padded to 4)
  tsg::DevBuf<int32_t> conn;            // [E][conn_stride]: node | (dof-mask bits << 28)
  tsg::DevBuf<int32_t> conn3;           // [E][12|8]: 3*node per local node, then dof-mask word
  tsg::DevBuf<unsigned char> coef;      // [E][12] of T: b_1,b_2,b_3, lp, mp, 0
  tsg::DevBuf<unsigned char> mask;      // [3N] uint8 (empty if unconstrained)
  tsg::DevBuf<int32_t> masked_dofs;     // constrained dof indices (identity rows)
  int32_t n_masked_dofs = 0;
  tsg::HostVec<double> coef64;          // host [E][12]: b (9), lambda*V, mu*V, V  (setup only)
  tsg::HostVec<int32_t> host_conn;      // host [E][npe] (setup only)
  tsg::HostVec<int32_t> elem_order;     // host [E]: caller's element id at each sweep position
  std::vector<uint8_t> host_mask;       // host [3N]
  std::unique_ptr<EbeColorPlan> color;  // greedy element coloring (deterministic sweep)
  bool deterministic = false;           // colored sweep: order-fixed sums, batch-independent bits
  int32_t group_split = 0;              // elements [0, split) = group 0 (partition boundary), rest group 1
  std::unique_ptr<EbePairPlan> pair;    // face-sharing pairs (kernels 6 = default, 7)
  std::unique_ptr<EbeFanPlan> fan;      // edge fans (kernel 8, tet10)
  int kernel = 6;  // 2 pipelined generic, 3 pipelined batch-specialised, 6 = 7 face pairs (default),
                   // 8 edge fans; each falls back to 3, then 2, for batch widths it does not cover;
                   // `deterministic` overrides all of them with the colored sweep
  mutable std::mutex host_mu;            // guards the host-entry staging buffers (and `stream`)
  mutable std::unique_ptr<EbeStreamPlan> stream;  // built at the first pinned-host apply
  mutable tsg::DevBuf<unsigned char> stage_u, stage_f;
  bool timing = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.f;
  ~ts_ebe();
};

namespace tsg {
// Launch facts of one persistent sweep kernel on the CURRENT device: SM count and
// resident blocks per SM at `smem` bytes of dynamic shared memory. The shared-memory
// opt-in is a per-device function attribute, so it is set (and the occupancy
// queried) once per device and per larger size, under a lock (callers may run on
// several host threads, e.g. the in-process ranks of the partitioned tests).
struct KernelFit {
  int sms = 0;
  int per_sm = 0;
};
template <auto Kernel>
KernelFit kernel_fit(int threads, size_t smem) {
  constexpr int kMaxDevices = 64;
  static std::mutex mu;
  static KernelFit fit[kMaxDevices];
  static size_t configured[kMaxDevices] = {};
  int dev = 0;
  TS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("kernel_fit: device ordinal out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!fit[dev].sms || smem > configured[dev]) {
    TS_CUDA(cudaDeviceGetAttribute(&fit[dev].sms, cudaDevAttrMultiProcessorCount, dev));
    if (smem > configured[dev]) {
      TS_CUDA(cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      configured[dev] = smem;
    }
    TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit[dev].per_sm, Kernel, threads, configured[dev]));
  }
  return fit[dev];
}

// Units per launch of a persistent unit sweep (ebe_pair.cu): statically strided sweeps split
// long sweeps into launches of a bounded number of grid strides (TSGPU_EBE_PAIR_STRIDES);
// the pair sweep's dynamic schedule (pair_dynamic) runs one launch
int64_t strided_launch_units(int64_t units_per_stride, int64_t units);
int64_t pair_launch_units(int64_t units_per_stride, int64_t units);
// fan sweep (ebe_fan.cu): units [q0, q1) / an element group; false if `batch` is not covered
bool ebe_fan_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t q0,
                         int32_t q1);
bool ebe_fan_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part);
int ebe_fan_launches(const ts_ebe& op, int32_t batch);
void build_fan_plan(ts_ebe& op, const Mesh& m, const HostVec<int32_t>& conn_words, int cs,
                    const HostVec<double>& coef64, bool fp32);
// the active unit sweep (fans, else pairs) over its units [q0, q1); unit count of the active plan
bool ebe_unit_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t q0,
                          int32_t q1);
int32_t ebe_unit_count(const ts_ebe& op);
// pair sweep over units [p0, p1) (no init); false if the pair kernel does not cover `batch`
bool ebe_pair_apply_range(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int32_t p0,
                          int32_t p1);
// f = A u with HOST u, f: H2D of u, the sweep and D2H of f overlapped chunk by chunk when
// the buffers are pinned and the operator has a streamable schedule, else copy-apply-copy
void ebe_apply_host(const ts_ebe& op, const void* u, void* f, int32_t batch);
// f = A u on device pointers (EbeOperator::apply, ebe_operator.hpp:90-134)
void ebe_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s);
// inverse nodal diagonal blocks, fp64 math, rounded to prec (ebe_operator.hpp:288-313);
// writes a DEVICE array [n_nodes][9] of the operator precision
void ebe_block_jacobi(const ts_ebe& op, void* inv_dev, cudaStream_t s);
// the two halves of ebe_block_jacobi: fp64 nodal diagonal blocks [n][9] of sum_e K_e,
// then invert_node_block per node (block_jacobi.hpp:45-66) rounded to prec
void ebe_diag_blocks(const ts_ebe& op, double* diag_dev, cudaStream_t s);
void bj_invert(const double* diag_dev, const uint8_t* mask_dev, int32_t n, int prec, void* inv_dev, cudaStream_t s);
// colored deterministic sweep (ebe_color.cu) over element range part (-1 all, 0 boundary, 1 interior)
void ebe_color_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part);
// builds the coloring once (host, setup data); on = deterministic sweeps from now on
void ebe_set_deterministic(ts_ebe& op, bool on);
// element-group sweep of a partitioned operator (part -1 all, 0 boundary, 1 interior)
void ebe_apply_part(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part, bool init);
// kernel launches of one device apply of `batch` cases (init + sweep); pair sweep alone: -1 = not covered
int ebe_launches_per_apply(const ts_ebe& op, int32_t batch);
int ebe_pair_launches(const ts_ebe& op, int32_t batch);
// pair sweep (ebe_pair.cu); false when no instance covers this batch width
bool pair_dynamic();  // TSGPU_EBE_DYN: pair units taken in warp chunks from a counter
// f (its masked-identity start already written) += K u over the pair sweep (part -1: whole, one
// element group, + the constrained dofs' p.p; 0 / 1: that element group only), plus the inner
// PCG's gamma partials (p, Ap) in dpart[block][3][batch] (fp32 tet10, r = 8 / 16, dynamic schedule);
// returns the partial rows written, or -1 (nothing launched)
int ebe_pair_apply_dots(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, double* dpart,
                        int part = -1);
// sum over the constrained dofs `dofs` of p^2 per column into dpart rows (at most rows_left); rows written
int ebe_masked_pp(const int32_t* dofs, int32_t n, const float* p, int32_t batch, cudaStream_t s, double* dpart,
                  int rows_left);
bool ebe_pair_apply(const ts_ebe& op, const void* u, void* f, int32_t batch, cudaStream_t s, int part);
// face-pair topology of an element order (greedy matching result), shareable between the
// level set's tet10 operators, which use the same mesh and element order
struct PairTopology {
  int64_t n_elems = -1;
  int32_t group_split = -1;
  std::vector<int32_t> mate;
  std::vector<int8_t> mate_k;
  std::vector<int32_t> units;
  int32_t split = 0;
};
void build_pair_plan(ts_ebe& op, const Mesh& m, const HostVec<int32_t>& conn_words, int cs,
                     const HostVec<double>& coef64, bool fp32, PairTopology* topo = nullptr);
// elem_group (nullable, [E] in {0,1}): group-0 elements sweep separately (boundary first);
// kernel_override >= 0 fixes the sweep kernel (and so which plans are built);
// element_order (nullable): empty -> receives the Morton order, filled -> reused
ts_ebe* ebe_create(const Mesh& m, int order, int32_t n_mat, const double* lambda,
                   const double* mu, const uint8_t* dof_mask, int prec, const uint8_t* elem_group = nullptr,
                   int kernel_override = -1, std::vector<int32_t>* element_order = nullptr,
                   PairTopology* pair_topology = nullptr);
}  // namespace tsg
