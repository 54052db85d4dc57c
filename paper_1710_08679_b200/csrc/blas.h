// blas.h — device vector / transfer / small-operator kernels of the solve path.
// All vectors are [node][axis][case] with `batch` cases (vector_batch.hpp:12-28).
#pragma once
#include "comm.h"
#include "ts_common.h"

namespace tsg {

// fixed reduction geometry: deterministic per-column fp64 sums
constexpr int kRedBlocks = 1184;   // reduction grid cap: 8 x 148 SMs (big levels)
constexpr int kRedMinBlocks = 148; // floor: one block per SM (small levels; fewer partials to finalize)
constexpr int kRedThreads = 256;

// Per-column solver scalars living on the device (one array of `batch` each).
struct ColScalars {
  DevBuf<double> buf;
  int32_t batch = 0;
  enum { RN2, EN2, RHO_A, RHO_B, BETA, GAMMA, ALPHA, PP, QQ, FN2, ZQ, GPREV, TMP, N_ };
  void ensure(int32_t b) {
    if (b != batch) {
      buf.alloc(static_cast<size_t>(N_) * b);
      batch = b;
    }
  }
  double* operator[](int k) const { return buf.get() + static_cast<size_t>(k) * batch; }
};

// status read back by the host once per iteration
struct PcgStatus {
  double ratio;       // max_b num/den (pcg.hpp:32-42)
  int stagnated;      // pcg.hpp:99-104
  int breakdown_col;  // first column with (p,Ap) <= 0 and no stagnation, else -1
  int nonfinite;
  int need_full;      // fused gamma partials hit the (p,Ap) <= 0 branch: rerun it with the full dot pass
};

// Collective hooks of a distributed solve (comm.h); null on one device.
struct Comm;

struct Workspace {
  DevBuf<double> partial;  // [kRedBlocks][4][batch]
  DevBuf<double> summed;   // [4][batch] per-rank column sums (distributed)
  Comm* comm = nullptr;             // set: reductions are all-reduced across ranks
  const uint8_t* owned = nullptr;   // set: per-node ownership flags of the current level's vectors
  DevBuf<PcgStatus> status;
  PcgStatus* host_status = nullptr;  // pinned
  // (M^-1 e, e) partials left by the last pcg_init / pcg_update (slot nd-1), consumed by pcg_rho
  const double* last_p = nullptr;
  int last_nblk = 0, last_nd = 0;
  int nblk = kRedBlocks;  // grid of the last reduction launch (red_grid)
  void ensure(int32_t batch);
  ~Workspace();
};

// ---- reductions ------------------------------------------------------------
// out[b] = (x0,y0)_b and, when x1 != null, out[batch + b] = (x1,y1)_b; fp64 accumulation
template <typename T>
void dot2(const T* x0, const T* y0, const T* x1, const T* y1, int64_t ndof, int32_t batch, double* out,
          Workspace& ws, cudaStream_t s);

// ---- inner PCG steps (pcg.hpp:52-124), T = float | double --------------------
// rho_a = (M^-1 e, e) from the partials of the last pcg_init / pcg_update;
// beta = first ? 0 : (rho_b != 0 ? rho_a / rho_b : 0)
void pcg_rho(int32_t batch, bool first, const ColScalars& cs, Workspace& ws, cudaStream_t s);
// p = M^-1 e + beta p  (first: p = M^-1 e); q_init (optional): masked identity of the new p
// (zeros where mask is null), the starting value of the following EBE product;
// u_pending (optional, not on the first iteration): first u += alpha p with the OLD p
// (the update pass defers it)
template <typename T>
void pcg_direction(const T* inv, const T* e, T* p, int32_t n_nodes, int32_t batch, bool first,
                   const ColScalars& cs, cudaStream_t s, T* q_init = nullptr, const uint8_t* mask = nullptr,
                   T* u_pending = nullptr);
// u += alpha p: the deferred update of the last iteration, when the loop ends after an update
template <typename T>
void pcg_apply_pending(T* u, const T* p, int32_t n_nodes, int32_t batch, const ColScalars& cs, cudaStream_t s);
// gamma = (p,q), plus ||p||^2, ||q||^2; alpha + stagnation/breakdown flags
template <typename T>
void pcg_gamma(const T* p, const T* q, int32_t n_nodes, int32_t batch, const ColScalars& cs, Workspace& ws,
               cudaStream_t s);
// unless stagnated/broken: e -= alpha q ; en2 = ||e||^2 ; ratio; also the (M^-1 e, e)
// partials of the next iteration (pcg_rho). The matching u += alpha p is left pending
// (pcg_direction's u_pending / pcg_apply_pending).
template <typename T>
void pcg_update(const T* inv, T* e, const T* q, int32_t n_nodes, int32_t batch, const ColScalars& cs,
                Workspace& ws, cudaStream_t s);
// e = r - Au (Au in e on entry); rn2 = ||r||^2, en2 = ||e||^2, ratio; (M^-1 e, e) partials
template <typename T>
void pcg_init(const T* inv, const T* r, T* e, int32_t n_nodes, int32_t batch, const ColScalars& cs, Workspace& ws,
              cudaStream_t s);

// ---- outer CG steps (adaptive_cg.hpp:126-233), fp64 -------------------------
// r = f - r (K u in r on entry); rn2 = ||r||^2 ; ratio vs fn2
void cg_true_residual(const double* f, double* r, int32_t n_nodes, int32_t batch, const ColScalars& cs,
                      Workspace& ws, cudaStream_t s);
// beta = gprev != 0 ? -(z,q)/gprev : 0 ; p = z + beta p  (first: p = z)
void cg_direction(const double* z, const double* q, double* p, int32_t n_nodes, int32_t batch, bool first,
                  const ColScalars& cs, Workspace& ws, cudaStream_t s);
// rho = (z,r), gamma = (p,q); alpha with breakdown check; gprev = gamma
void cg_alpha(const double* z, const double* r, const double* p, const double* q, int32_t n_nodes,
              int32_t batch, const ColScalars& cs, Workspace& ws, cudaStream_t s);
// r -= alpha q ; u += alpha p ; rn2 ; ratio vs fn2
void cg_update(double* r, double* u, const double* p, const double* q, int32_t n_nodes, int32_t batch,
               const ColScalars& cs, Workspace& ws, cudaStream_t s);

// ---- small operators ---------------------------------------------------------
// z = M^-1 r per node, fp64 math rounded to T (block_jacobi.hpp:22-38)
template <typename T>
void bj_apply(const T* inv, const T* r, T* z, int32_t n_nodes, int32_t batch, cudaStream_t s);
// f = A u, 3x3 float blocks, fp64 row accumulation (block_csr.hpp:33-69)
void bcsr_apply_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n,
                    const float* u, float* f, int32_t batch, cudaStream_t s, int64_t nnz = -1);
// the assembled level-1 operator (fp32 blocks, fp32 accumulation): y = K1 x
// rows (nullable): apply only these n rows (row ids) instead of rows [0, n)
// level-1 product q = K1 p that also leaves the gamma pass's partials ((p,q), (p,p), (q,q) per
// column, reduce_pass layout) in ws.partial / ws.nblk; false (nothing launched) when it does not
// apply (unstaged width, distributed workspace)
bool bcsr_rows_f32_gamma(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n,
                         const float* p, float* q, int32_t batch, cudaStream_t s, int64_t nnz, Workspace& ws,
                         const uint8_t* rowsel = nullptr);
// the level-2 product (fp64 row sums) with gamma's partials, as bcsr_rows_f32_gamma; one device / replicated only
bool bcsr_apply_f32_gamma(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n,
                          const float* p, float* q, int32_t batch, cudaStream_t s, int64_t nnz, Workspace& ws);
// partitioned: rowsel[r] = 1 for the rows the fused product counts; the rest of this rank's rows (its
// owned interface rows, complete after the exchange) are added by rows_dots_append
void rows_dots_append(const float* p, const float* q, const int32_t* rows, int32_t n, int32_t batch, cudaStream_t s,
                      Workspace& ws);
// the gamma finalize (alpha, breakdown / stagnation) from partials already in ws; partial_pq_only:
// the partials hold (p,q) alone (element-wise products), so a column with (p,q) <= 0 sets
// need_full instead of deciding stagnation / breakdown (pcg_update then leaves e alone)
template <typename T>
void pcg_gamma_final(int32_t batch, const ColScalars& cs, Workspace& ws, cudaStream_t s, bool partial_pq_only = false);
// whether whole-range products of `batch` cases take the warp-staged kernel
bool bcsr_rows_staged_ok(int32_t batch);
// nnz (the blocks / column entries stored; -1 = unknown) enables the warp-staged kernel for
// whole-range products (rows == nullptr)
void bcsr_rows_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n, const float* u,
                   float* f, int32_t batch, cudaStream_t s, const int32_t* rows = nullptr, int64_t nnz = -1);
// casts (cast_batch, vector_batch.hpp:43-49)
void cast_d2f(const double* x, float* y, int64_t n, cudaStream_t s);
void cast_f2d(const float* x, double* y, int64_t n, cudaStream_t s);
// zero constrained dofs (zero_masked, vector_batch.hpp:109-119)
void zero_masked_f32(float* x, const uint8_t* mask, int64_t ndof, int32_t batch, cudaStream_t s);
// geometric P1->P2: vertex rows copy, edge rows 0.5 a + 0.5 b (prolongation.hpp:25-40,67-98)
void p1_apply(const float* coarse, float* fine, const int32_t* edge_ends, int32_t n_vert, int32_t n_fine,
              const uint8_t* fine_mask, int32_t batch, cudaStream_t s);
// restriction P1^T as a gather over the transpose in ascending fine order (bit-exact
// with the reference's serial scatter, prolongation.hpp:44-61), then zero_masked
// (owned: nullable per-vertex flags; a partition counts the vertex's own row only on its owner)
void p1_restrict(const float* fine, float* coarse, const int32_t* t_ptr, const int32_t* t_idx,
                 int32_t n_vert, const uint8_t* coarse_mask, int32_t batch, cudaStream_t s,
                 const uint8_t* owned = nullptr);
// aggregation P2: fine = coarse[agg]; restrict = ascending-member sums
void p2_apply(const float* coarse, float* fine, const int32_t* agg, int32_t n_fine, const uint8_t* fine_mask,
              int32_t batch, cudaStream_t s);
void p2_restrict(const float* fine, float* coarse, const int32_t* a_ptr, const int32_t* a_idx, int32_t n_coarse,
                 const uint8_t* coarse_mask, int32_t batch, cudaStream_t s);

}  // namespace tsg
