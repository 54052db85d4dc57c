// ops.cu — the reference's standalone solve-path operators behind the C ABI:
// BlockCsrMatrix<T>::apply (block_csr.hpp:33-69), BlockJacobi<T>::apply
// (block_jacobi.hpp:22-38) and its extraction from a block-CSR matrix
// (:72-85), Prolongation::apply / restrict_to_coarse (prolongation.hpp:25-61)
// and build_geometric_prolongation (:67-98), inner_pcg on any of the
// operators (pcg.hpp:52-124), EbeOperator::element_matrix (ebe_operator.hpp:
// 78-87) and assemble_bcsr (:230-284), and the per-column vector operations
// of vector_batch.hpp:43-119.
//
// The multigrid solve (solver.cu) runs fused, level-specialised versions of
// the same kernels; these entries give a reference caller the operators one
// at a time (the drop-in headers include/tetsolve/*.hpp sit on them). Every
// arithmetic step runs on the device; host code here only validates, builds
// index structures (transposes, the assembly pattern) and moves buffers.
//
// Rounding: where the reference's result is exactly defined by its operation
// order (prolongation and column updates in T, BCSR rows accumulated in fp64
// in stored-block order), the kernels use the same order with explicit
// round-to-nearest intrinsics (no FMA contraction), so they agree bit for bit.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "blas.h"
#include "ebe.h"
#include "element_kernels.cuh"
#include "setup.h"
#include "solver_core.h"

// ---------------------------------------------------------------- handles
struct ts_bcsr {
  int prec = 32;
  int32_t n = 0;
  int64_t nnzb = 0;
  tsg::DevBuf<int32_t> row_ptr, col_idx;
  tsg::DevBuf<unsigned char> blocks;  // [nnzb][9] of T
  std::vector<int32_t> h_row_ptr, h_col_idx;
};

struct ts_bj {
  int prec = 32;
  int32_t n = 0;
  tsg::DevBuf<unsigned char> inv;  // [n][9] of T
};

struct ts_prolong {
  int32_t n_fine = 0, n_coarse = 0;
  tsg::DevBuf<int32_t> row_ptr, cols;     // per fine node
  tsg::DevBuf<double> weights;
  tsg::DevBuf<int32_t> t_ptr, t_rows;     // transpose: per coarse node, fine rows ascending
  tsg::DevBuf<double> t_weights;
};

namespace tsg {
namespace {

// exact-rounding helpers: one rounding per operation, as the reference's scalar loops
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }

// BlockCsrMatrix<T>::apply: one thread per (block row, case); fp64 row accumulators,
// a[b] += b0 u0 + b1 u1 + b2 u2 per stored block in stored order (block_csr.hpp:40-54)
template <typename T>
__global__ void k_bcsr_apply(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                             const T* __restrict__ blocks, int32_t n, const T* __restrict__ u, T* __restrict__ f,
                             int32_t B) {
  const int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (it >= int64_t(n) * B) return;
  const int64_t r = it / B;
  const int b = static_cast<int>(it - r * B);
  double a[3] = {0.0, 0.0, 0.0};
  for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
    const T* blk = blocks + 9 * int64_t(e);
    const T* uc = u + 3 * int64_t(col_idx[e]) * B + b;
    const double u0 = double(uc[0]), u1 = double(uc[B]), u2 = double(uc[2 * B]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double s = __dadd_rn(__dadd_rn(__dmul_rn(double(blk[3 * i]), u0), __dmul_rn(double(blk[3 * i + 1]), u1)),
                                 __dmul_rn(double(blk[3 * i + 2]), u2));
      a[i] = __dadd_rn(a[i], s);
    }
  }
  T* fr = f + 3 * r * B + b;
#pragma unroll
  for (int i = 0; i < 3; ++i) fr[i * B] = static_cast<T>(a[i]);
}

// diagonal blocks of a block-CSR matrix as fp64 (extract_block_jacobi(BCSR), block_jacobi.hpp:72-85);
// rows without a stored diagonal block give a zero block (singular -> ValidationError)
template <typename T>
__global__ void k_bcsr_diag(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                            const T* __restrict__ blocks, int32_t n, double* __restrict__ diag) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double d[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e)
    if (col_idx[e] == r) {
      for (int q = 0; q < 9; ++q) d[q] = double(blocks[9 * int64_t(e) + q]);
      break;
    }
  for (int q = 0; q < 9; ++q) diag[9 * r + q] = d[q];
}

// Prolongation::apply: out = 0; out += (T)w * in per stored entry, in T (prolongation.hpp:31-40)
template <typename T>
__global__ void k_prolong(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                          const double* __restrict__ w, int32_t n_out, const T* __restrict__ in, T* __restrict__ out,
                          int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = 3 * int64_t(n_out) * B;
  if (i >= len) return;
  const int64_t node = i / (3 * int64_t(B));
  const int64_t rem = i - node * 3 * B;  // axis * B + b
  T v = T(0);
  for (int32_t k = ptr[node]; k < ptr[node + 1]; ++k)
    v = radd(v, rmul(static_cast<T>(w[k]), in[3 * int64_t(idx[k]) * B + rem]));
  out[i] = v;
}

// y = A x for one operand of a kernel on a single (unit) vector: columns of K_e
// (ebe_operator.hpp:78-87 element_matrix); K_e is symmetric, so column j = row j.
// rec: b_1..b_3 (9), lambda V, mu V (the operator's fp64 setup record)
template <int NPE>
__device__ void element_column(const double* __restrict__ rec, int j, double (&col)[NPE][3]) {
  double b[3][3];
  for (int k = 0; k < 3; ++k)
    for (int d = 0; d < 3; ++d) b[k][d] = rec[3 * k + d];
  const double scale = NPE == 10 ? 1.0 / 20.0 : 1.0;
  const double lp = rec[9] * scale, mp = rec[10] * scale;
  double uu[NPE][3];
  for (int a = 0; a < NPE; ++a)
    for (int c = 0; c < 3; ++c) uu[a][c] = (3 * a + c == j) ? 1.0 : 0.0;
  if constexpr (NPE == 10) tet10_product<double>(uu, b, lp, mp, col);
  else tet4_product<double>(uu, b, lp, mp, col);
}

template <int NPE>
__global__ void k_element_matrix(const double* __restrict__ rec, double* __restrict__ k) {
  const int j = threadIdx.x;
  if (j >= 3 * NPE) return;
  double col[NPE][3];
  element_column<NPE>(rec, j, col);
  for (int a = 0; a < NPE; ++a)
    for (int c = 0; c < 3; ++c) k[(3 * a + c) * 3 * NPE + j] = col[a][c];  // row-major, index 3 node + axis
}

// assemble_bcsr (ebe_operator.hpp:230-284): one thread per block row; the row's
// incident elements in ascending (caller) element order, the rows 3a+i of K_e by
// symmetry from the element product on unit vectors, accumulated in fp64 into the
// row's blocks (constrained rows / columns skipped), identity on constrained diagonals.
template <int NPE>
__global__ void k_assemble_rows(const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc_pos,
                                const int32_t* __restrict__ conn, const double* __restrict__ c64,
                                const uint8_t* __restrict__ mask, const int32_t* __restrict__ row_ptr,
                                const int32_t* __restrict__ col_idx, int32_t n, double* __restrict__ acc) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t rb = row_ptr[r], re = row_ptr[r + 1];
  auto entry = [&](int32_t c) {
    int32_t lo = rb, hi = re;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (col_idx[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  for (int64_t k = inc_ptr[r]; k < inc_ptr[r + 1]; ++k) {
    const int64_t pos = inc_pos[k];
    const int32_t* t = conn + NPE * pos;
    int a = 0;
    while (t[a] != r) ++a;
    for (int i = 0; i < 3; ++i) {
      if (mask && mask[3 * r + i]) continue;
      double row[NPE][3];
      element_column<NPE>(c64 + 12 * pos, 3 * a + i, row);
      for (int bn = 0; bn < NPE; ++bn) {
        const int32_t gb = t[bn];
        double* blk = acc + 9 * int64_t(entry(gb));
        for (int j = 0; j < 3; ++j) {
          if (mask && mask[3 * int64_t(gb) + j]) continue;
          blk[3 * i + j] += row[bn][j];
        }
      }
    }
  }
  if (mask) {
    double* d = acc + 9 * int64_t(entry(static_cast<int32_t>(r)));
    for (int i = 0; i < 3; ++i)
      if (mask[3 * r + i]) d[4 * i] = 1.0;
  }
}

template <typename T>
__global__ void k_cast_blocks(const double* __restrict__ x, T* __restrict__ y, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = static_cast<T>(x[i]);
}

// ---- per-column vector ops (vector_batch.hpp:43-119) ----
// dot_columns: one block per column, fixed-order fp64 sums (strided partials, then a tree)
template <typename T>
__global__ void k_dot_columns(const T* __restrict__ x, const T* __restrict__ y, int64_t ndof, int32_t B,
                              double* __restrict__ out) {
  __shared__ double sm[256];
  const int b = blockIdx.x;
  double acc = 0.0;
  for (int64_t d = threadIdx.x; d < ndof; d += blockDim.x) acc += double(x[d * B + b]) * double(y[d * B + b]);
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = sm[0];
}
// y += (T)alpha[b] x
template <typename T>
__global__ void k_axpy_columns(const double* __restrict__ alpha, const T* __restrict__ x, T* __restrict__ y,
                               int64_t len, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) y[i] = radd(y[i], rmul(static_cast<T>(alpha[i % B]), x[i]));
}
// p = z + (T)beta[b] p
template <typename T>
__global__ void k_xpby_columns(const T* __restrict__ z, const double* __restrict__ beta, T* __restrict__ p,
                               int64_t len, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) p[i] = radd(z[i], rmul(static_cast<T>(beta[i % B]), p[i]));
}
template <typename T>
__global__ void k_sub_columns(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, int64_t len) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) out[i] = rsub(a[i], b[i]);
}
template <typename T>
__global__ void k_zero_masked(T* __restrict__ x, const uint8_t* __restrict__ mask, int64_t len, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len && mask[i / B]) x[i] = T(0);
}
template <typename From, typename To>
__global__ void k_cast(const From* __restrict__ x, To* __restrict__ y, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = static_cast<To>(x[i]);
}

size_t tsize(int prec) { return prec == 32 ? 4 : 8; }
void check_prec(int prec, const char* what) {
  if (prec != 32 && prec != 64) validation(std::string(what) + ": precision must be 32 or 64");
}

void bcsr_apply_dev(const ts_bcsr& a, const void* u, void* f, int32_t B, cudaStream_t s) {
  if (B < 1) validation("bcsr apply: batch must be >= 1");
  if (a.n == 0) return;
  const unsigned g = grid_for(int64_t(a.n) * B, 256);
  if (a.prec == 32)
    k_bcsr_apply<float><<<g, 256, 0, s>>>(a.row_ptr.get(), a.col_idx.get(),
                                          reinterpret_cast<const float*>(a.blocks.get()), a.n,
                                          static_cast<const float*>(u), static_cast<float*>(f), B);
  else
    k_bcsr_apply<double><<<g, 256, 0, s>>>(a.row_ptr.get(), a.col_idx.get(),
                                           reinterpret_cast<const double*>(a.blocks.get()), a.n,
                                           static_cast<const double*>(u), static_cast<double*>(f), B);
  TS_CUDA_LAUNCH();
}

void bj_apply_dev(const ts_bj& m, const void* r, void* z, int32_t B, cudaStream_t s) {
  if (B < 1) validation("block jacobi apply: batch must be >= 1");
  if (m.n == 0) return;
  if (m.prec == 32)
    bj_apply<float>(reinterpret_cast<const float*>(m.inv.get()), static_cast<const float*>(r), static_cast<float*>(z),
                    m.n, B, s);
  else
    bj_apply<double>(reinterpret_cast<const double*>(m.inv.get()), static_cast<const double*>(r),
                     static_cast<double*>(z), m.n, B, s);
}

void prolong_dev(const ts_prolong& p, int prec, bool restrict_, const void* in, void* out, int32_t B,
                 cudaStream_t s) {
  check_prec(prec, "prolongation");
  if (B < 1) validation("prolongation: batch must be >= 1");
  const int32_t n_out = restrict_ ? p.n_coarse : p.n_fine;
  if (n_out == 0) return;
  const int32_t* ptr = restrict_ ? p.t_ptr.get() : p.row_ptr.get();
  const int32_t* idx = restrict_ ? p.t_rows.get() : p.cols.get();
  const double* w = restrict_ ? p.t_weights.get() : p.weights.get();
  const unsigned g = grid_for(3 * int64_t(n_out) * B, 256);
  if (prec == 32)
    k_prolong<float><<<g, 256, 0, s>>>(ptr, idx, w, n_out, static_cast<const float*>(in), static_cast<float*>(out), B);
  else
    k_prolong<double><<<g, 256, 0, s>>>(ptr, idx, w, n_out, static_cast<const double*>(in), static_cast<double*>(out),
                                        B);
  TS_CUDA_LAUNCH();
}

// run a device routine on host buffers: inputs up, outputs down (synchronous)
struct Staged {
  std::vector<DevBuf<unsigned char>> bufs;
  void* in(const void* h, size_t bytes) {
    bufs.emplace_back(bytes);
    if (bytes) TS_CUDA(cudaMemcpy(bufs.back().get(), h, bytes, cudaMemcpyHostToDevice));
    return bufs.back().get();
  }
  void* out(size_t bytes) {
    bufs.emplace_back(bytes);
    return bufs.back().get();
  }
};
void down(void* h, const void* d, size_t bytes) {
  if (bytes) TS_CUDA(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost));
}

// inner_pcg (pcg.hpp:52-124) on device vectors through the shared core loop
template <typename T>
core::InnerStats inner_pcg_dev(int kind, const void* op, const ts_bj& m, const T* r, T* u, int32_t n, int32_t B,
                               double tol, int max_iter, cudaStream_t s) {
  const size_t len = 3 * size_t(n) * B;
  DevBuf<T> e(len), p(len), q(len);
  ColScalars cs;
  cs.ensure(B);
  Workspace ws;
  ws.ensure(B);
  auto A = [&](const T* x, T* y, bool) {
    if (kind == 0) ebe_apply(*static_cast<const ts_ebe*>(op), x, y, B, s);
    else bcsr_apply_dev(*static_cast<const ts_bcsr*>(op), x, y, B, s);
  };
  const core::InnerStats st = core::inner_pcg<T>(A, reinterpret_cast<const T*>(m.inv.get()), r, u, n, B, tol,
                                                 max_iter, e.get(), p.get(), q.get(), cs, ws, s);
  TS_CUDA(cudaStreamSynchronize(s));
  return st;
}

void op_shape(int kind, const void* op, int32_t* n, int* prec) {
  if (kind == 0) {
    const auto* k = static_cast<const ts_ebe*>(op);
    *n = k->n_nodes;
    *prec = k->prec;
  } else if (kind == 1) {
    const auto* a = static_cast<const ts_bcsr*>(op);
    *n = a->n;
    *prec = a->prec;
  } else {
    validation("inner_pcg: operator kind must be 0 (EbeOperator) or 1 (BlockCsrMatrix)");
  }
}

}  // namespace
}  // namespace tsg

#define TS_API_BEGIN try {
#define TS_API_END                              \
  }                                             \
  catch (const tsg::Error& e) {                 \
    tsg::set_last_error(e.what());              \
    return e.code;                              \
  }                                             \
  catch (const std::bad_alloc&) {               \
    tsg::set_last_error("out of host memory");  \
    return TS_ERR_VALIDATION;                   \
  }                                             \
  catch (const std::exception& e) {             \
    tsg::set_last_error(e.what());              \
    return TS_ERR_VALIDATION;                   \
  }                                             \
  return TS_OK;

using tsg::validation;

extern "C" {

// ------------------------------------------------------------ block CSR
ts_status ts_bcsr_create(int32_t n_block_rows, const int32_t* row_ptr, const int32_t* col_idx, const void* blocks,
                         int32_t prec, ts_bcsr** out) {
  TS_API_BEGIN
  if (!out || !row_ptr || n_block_rows < 0) validation("bcsr: null argument");
  tsg::check_prec(prec, "bcsr");
  tsg::require_device();
  if (row_ptr[0] != 0) validation("bcsr: row_ptr[0] must be 0");
  for (int32_t r = 0; r < n_block_rows; ++r)
    if (row_ptr[r + 1] < row_ptr[r]) validation("bcsr: row_ptr must be non-decreasing");
  const int64_t nnzb = row_ptr[n_block_rows];
  if (nnzb > 0 && (!col_idx || !blocks)) validation("bcsr: null argument");
  for (int32_t r = 0; r < n_block_rows; ++r)
    for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      if (col_idx[e] < 0 || col_idx[e] >= n_block_rows)
        validation("bcsr: column index out of range in block row " + std::to_string(r));
      if (e > row_ptr[r] && col_idx[e] <= col_idx[e - 1])  // block_csr.hpp:14 invariant
        validation("bcsr: column indices must be strictly increasing in block row " + std::to_string(r));
    }
  auto a = std::make_unique<ts_bcsr>();
  a->prec = prec;
  a->n = n_block_rows;
  a->nnzb = nnzb;
  a->h_row_ptr.assign(row_ptr, row_ptr + n_block_rows + 1);
  a->h_col_idx.assign(col_idx, col_idx + nnzb);
  a->row_ptr.upload(a->h_row_ptr);
  a->col_idx.upload(a->h_col_idx);
  a->blocks.upload(static_cast<const unsigned char*>(blocks), size_t(nnzb) * 9 * tsg::tsize(prec));
  TS_CUDA(cudaDeviceSynchronize());
  *out = a.release();
  TS_API_END
}

void ts_bcsr_destroy(ts_bcsr* a) { delete a; }

ts_status ts_bcsr_info(const ts_bcsr* a, int32_t* n_block_rows, int64_t* nnzb, int32_t* prec) {
  TS_API_BEGIN
  if (!a) validation("bcsr: null handle");
  if (n_block_rows) *n_block_rows = a->n;
  if (nnzb) *nnzb = a->nnzb;
  if (prec) *prec = a->prec;
  TS_API_END
}

ts_status ts_bcsr_apply(const ts_bcsr* a, const void* u, void* f, int32_t batch, void* stream) {
  TS_API_BEGIN
  if (!a || !u || !f) validation("bcsr apply: null argument");
  tsg::bcsr_apply_dev(*a, u, f, batch, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_bcsr_apply_host(const ts_bcsr* a, const void* u, void* f, int32_t batch) {
  TS_API_BEGIN
  if (!a || !u || !f) validation("bcsr apply: null argument");
  if (batch < 1) validation("bcsr apply: batch must be >= 1");
  const size_t bytes = 3 * size_t(a->n) * batch * tsg::tsize(a->prec);
  tsg::Staged st;
  void* du = st.in(u, bytes);
  void* df = st.out(bytes);
  tsg::bcsr_apply_dev(*a, du, df, batch, nullptr);
  tsg::down(f, df, bytes);
  TS_API_END
}

ts_status ts_bcsr_block_jacobi_host(const ts_bcsr* a, void* inv_blocks) {
  TS_API_BEGIN
  if (!a || !inv_blocks) validation("block jacobi: null argument");
  tsg::DevBuf<double> diag(9 * size_t(a->n));
  tsg::DevBuf<unsigned char> inv(9 * size_t(a->n) * tsg::tsize(a->prec));
  if (a->n > 0) {
    const unsigned g = tsg::grid_for(a->n, 128);
    if (a->prec == 32)
      tsg::k_bcsr_diag<float><<<g, 128>>>(a->row_ptr.get(), a->col_idx.get(),
                                          reinterpret_cast<const float*>(a->blocks.get()), a->n, diag.get());
    else
      tsg::k_bcsr_diag<double><<<g, 128>>>(a->row_ptr.get(), a->col_idx.get(),
                                           reinterpret_cast<const double*>(a->blocks.get()), a->n, diag.get());
    TS_CUDA_LAUNCH();
    tsg::bj_invert(diag.get(), nullptr, a->n, a->prec, inv.get(), nullptr);
  }
  tsg::down(inv_blocks, inv.get(), 9 * size_t(a->n) * tsg::tsize(a->prec));
  TS_API_END
}

// ------------------------------------------------------------ block Jacobi
ts_status ts_bj_create(int32_t n_nodes, const void* inv_blocks, int32_t prec, ts_bj** out) {
  TS_API_BEGIN
  if (!out || n_nodes < 0 || (n_nodes > 0 && !inv_blocks)) validation("block jacobi: null argument");
  tsg::check_prec(prec, "block jacobi");
  tsg::require_device();
  auto m = std::make_unique<ts_bj>();
  m->prec = prec;
  m->n = n_nodes;
  m->inv.upload(static_cast<const unsigned char*>(inv_blocks), 9 * size_t(n_nodes) * tsg::tsize(prec));
  TS_CUDA(cudaDeviceSynchronize());
  *out = m.release();
  TS_API_END
}

void ts_bj_destroy(ts_bj* m) { delete m; }

ts_status ts_bj_apply(const ts_bj* m, const void* r, void* z, int32_t batch, void* stream) {
  TS_API_BEGIN
  if (!m || !r || !z) validation("block jacobi apply: null argument");
  tsg::bj_apply_dev(*m, r, z, batch, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_bj_apply_host(const ts_bj* m, const void* r, void* z, int32_t batch) {
  TS_API_BEGIN
  if (!m || !r || !z) validation("block jacobi apply: null argument");
  if (batch < 1) validation("block jacobi apply: batch must be >= 1");
  const size_t bytes = 3 * size_t(m->n) * batch * tsg::tsize(m->prec);
  tsg::Staged st;
  void* dr = st.in(r, bytes);
  void* dz = st.out(bytes);
  tsg::bj_apply_dev(*m, dr, dz, batch, nullptr);
  tsg::down(z, dz, bytes);
  TS_API_END
}

// ------------------------------------------------------------ transfers
ts_status ts_prolong_create(int32_t n_fine, int32_t n_coarse, const int32_t* row_ptr, const int32_t* cols,
                            const double* weights, ts_prolong** out) {
  TS_API_BEGIN
  if (!out || !row_ptr || n_fine < 0 || n_coarse < 0) validation("prolongation: null argument");
  tsg::require_device();
  if (row_ptr[0] != 0) validation("prolongation: row_ptr[0] must be 0");
  for (int32_t r = 0; r < n_fine; ++r)
    if (row_ptr[r + 1] < row_ptr[r]) validation("prolongation: row_ptr must be non-decreasing");
  const int32_t nnz = row_ptr[n_fine];
  if (nnz > 0 && (!cols || !weights)) validation("prolongation: null argument");
  for (int32_t k = 0; k < nnz; ++k)
    if (cols[k] < 0 || cols[k] >= n_coarse) validation("prolongation: coarse index out of range");
  // transpose in ascending fine row: the reference's serial scatter order (prolongation.hpp:52-60)
  std::vector<int32_t> tptr(size_t(n_coarse) + 1, 0), trows(nnz);
  std::vector<double> tw(nnz);
  for (int32_t k = 0; k < nnz; ++k) ++tptr[cols[k] + 1];
  for (int32_t c = 0; c < n_coarse; ++c) tptr[c + 1] += tptr[c];
  std::vector<int32_t> cur(tptr.begin(), tptr.end() - 1);
  for (int32_t r = 0; r < n_fine; ++r)
    for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
      const int32_t q = cur[cols[k]]++;
      trows[q] = r;
      tw[q] = weights[k];
    }
  auto p = std::make_unique<ts_prolong>();
  p->n_fine = n_fine;
  p->n_coarse = n_coarse;
  p->row_ptr.upload(row_ptr, size_t(n_fine) + 1);
  p->cols.upload(cols, nnz);
  p->weights.upload(weights, nnz);
  p->t_ptr.upload(tptr);
  p->t_rows.upload(trows);
  p->t_weights.upload(tw);
  TS_CUDA(cudaDeviceSynchronize());
  *out = p.release();
  TS_API_END
}

void ts_prolong_destroy(ts_prolong* p) { delete p; }

ts_status ts_prolong_apply(const ts_prolong* p, int32_t prec, const void* coarse, void* fine, int32_t batch,
                           void* stream) {
  TS_API_BEGIN
  if (!p || !coarse || !fine) validation("prolongation apply: null argument");
  tsg::prolong_dev(*p, prec, false, coarse, fine, batch, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_prolong_restrict(const ts_prolong* p, int32_t prec, const void* fine, void* coarse, int32_t batch,
                              void* stream) {
  TS_API_BEGIN
  if (!p || !coarse || !fine) validation("prolongation restrict: null argument");
  tsg::prolong_dev(*p, prec, true, fine, coarse, batch, static_cast<cudaStream_t>(stream));
  TS_API_END
}

ts_status ts_prolong_apply_host(const ts_prolong* p, int32_t prec, int32_t restrict_to_coarse, const void* in,
                                void* out, int32_t batch) {
  TS_API_BEGIN
  if (!p || !in || !out) validation("prolongation: null argument");
  tsg::check_prec(prec, "prolongation");
  if (batch < 1) validation("prolongation: batch must be >= 1");
  const size_t ts = tsg::tsize(prec);
  const size_t nin = restrict_to_coarse ? p->n_fine : p->n_coarse, nout = restrict_to_coarse ? p->n_coarse : p->n_fine;
  tsg::Staged st;
  void* di = st.in(in, 3 * nin * batch * ts);
  void* dout = st.out(3 * nout * batch * ts);
  tsg::prolong_dev(*p, prec, restrict_to_coarse != 0, di, dout, batch, nullptr);
  tsg::down(out, dout, 3 * nout * batch * ts);
  TS_API_END
}

// build_geometric_prolongation (prolongation.hpp:67-98): vertex rows identity, edge rows
// 0.5/0.5 on the endpoints; row_ptr [N+1], cols / weights [V + 2 (N - V)]
ts_status ts_geometric_prolongation(const ts_mesh* mesh, int32_t* row_ptr, int32_t* cols, double* weights) {
  TS_API_BEGIN
  if (!mesh || !row_ptr || !cols || !weights) validation("geometric prolongation: null argument");
  const tsg::Mesh& m = mesh->m;
  const int32_t N = m.n_nodes(), V = m.vertex_count;
  static constexpr int ee[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
  std::vector<int32_t> ends(2 * size_t(N - V), -1);
  for (int32_t e = 0; e < m.n_elems(); ++e) {
    const int32_t* t = m.tets10.data() + 10 * size_t(e);
    for (int q = 0; q < 6; ++q) {
      int32_t a = t[ee[q][0]], b = t[ee[q][1]];
      if (a > b) std::swap(a, b);
      const int32_t mid = t[4 + q];
      if (mid >= V) {
        ends[2 * size_t(mid - V)] = a;  // the mesh midpoint invariant: every copy carries the same ends
        ends[2 * size_t(mid - V) + 1] = b;
      }
    }
  }
  row_ptr[0] = 0;
  for (int32_t fn = 0; fn < N; ++fn) row_ptr[fn + 1] = row_ptr[fn] + (fn < V ? 1 : 2);
  for (int32_t fn = 0; fn < N; ++fn) {
    const int32_t k = row_ptr[fn];
    if (fn < V) {
      cols[k] = fn;
      weights[k] = 1.0;
    } else {
      if (ends[2 * size_t(fn - V)] < 0)
        validation("geometric prolongation: edge node " + std::to_string(fn) + " not present in edge map");
      cols[k] = ends[2 * size_t(fn - V)];
      cols[k + 1] = ends[2 * size_t(fn - V) + 1];
      weights[k] = weights[k + 1] = 0.5;
    }
  }
  TS_API_END
}

// ------------------------------------------------------------ inner PCG
ts_status ts_inner_pcg(int32_t kind, const void* op, const ts_bj* m, const void* r, void* u, int32_t n_nodes,
                       int32_t batch, double tol, int32_t max_iter, int32_t* iterations, int32_t* converged,
                       void* stream) {
  TS_API_BEGIN
  if (!op || !m || !r || !u) validation("inner_pcg: null argument");
  int32_t n = 0;
  int prec = 0;
  tsg::op_shape(kind, op, &n, &prec);
  if (n_nodes != n || m->n != n) validation("inner_pcg: dimension mismatch");
  if (m->prec != prec) validation("inner_pcg: preconditioner precision differs from the operator's");
  const auto s = static_cast<cudaStream_t>(stream);
  const tsg::core::InnerStats st =
      prec == 32 ? tsg::inner_pcg_dev<float>(kind, op, *m, static_cast<const float*>(r), static_cast<float*>(u), n,
                                             batch, tol, max_iter, s)
                 : tsg::inner_pcg_dev<double>(kind, op, *m, static_cast<const double*>(r), static_cast<double*>(u), n,
                                              batch, tol, max_iter, s);
  if (iterations) *iterations = st.iterations;
  if (converged) *converged = st.converged ? 1 : 0;
  TS_API_END
}

ts_status ts_inner_pcg_host(int32_t kind, const void* op, const ts_bj* m, const void* r, void* u, int32_t n_nodes,
                            int32_t batch, double tol, int32_t max_iter, int32_t* iterations, int32_t* converged) {
  TS_API_BEGIN
  if (!op || !m || !r || !u) validation("inner_pcg: null argument");
  int32_t n = 0;
  int prec = 0;
  tsg::op_shape(kind, op, &n, &prec);
  if (n_nodes != n) validation("inner_pcg: dimension mismatch");
  if (batch < 1) validation("inner_pcg: batch must be >= 1");
  const size_t bytes = 3 * size_t(n) * batch * tsg::tsize(prec);
  tsg::Staged st;
  const void* dr = st.in(r, bytes);
  void* du = st.in(u, bytes);
  ts_status rc = ts_inner_pcg(kind, op, m, dr, du, n_nodes, batch, tol, max_iter, iterations, converged, nullptr);
  if (rc != TS_OK) return rc;
  tsg::down(u, du, bytes);
  TS_API_END
}

// ------------------------------------------------------------ element matrices, assembly
ts_status ts_ebe_element_matrix(const ts_ebe* op, int32_t e, double* k) {
  TS_API_BEGIN
  if (!op || !k) validation("element_matrix: null argument");
  if (e < 0 || e >= op->n_elems) validation("element_matrix: element index out of range");
  if (op->coef64.size() != 12 * size_t(op->n_elems) || op->elem_order.size() != size_t(op->n_elems))
    validation("element_matrix: operator setup data released (level-set inner operators keep only device state)");
  // sweep position of caller element e
  const auto it = std::find(op->elem_order.begin(), op->elem_order.end(), e);
  const size_t pos = static_cast<size_t>(it - op->elem_order.begin());
  const int n = 3 * op->npe;
  tsg::DevBuf<double> rec(12), dk(size_t(n) * n);
  rec.upload(op->coef64.data() + 12 * pos, 12);
  if (op->npe == 10) tsg::k_element_matrix<10><<<1, 32>>>(rec.get(), dk.get());
  else tsg::k_element_matrix<4><<<1, 32>>>(rec.get(), dk.get());
  TS_CUDA_LAUNCH();
  tsg::down(k, dk.get(), size_t(n) * n * sizeof(double));
  TS_API_END
}

// assemble_bcsr: call with NULL arrays for *nnzb, then with row_ptr [n+1], col_idx [nnzb],
// blocks [nnzb][9] of the operator precision
ts_status ts_ebe_assemble_bcsr(const ts_ebe* op, int64_t* nnzb, int32_t* row_ptr, int32_t* col_idx, void* blocks) {
  TS_API_BEGIN
  if (!op || !nnzb) validation("assemble_bcsr: null argument");
  const int npe = op->npe;
  const int32_t n = op->n_nodes;
  const int64_t E = op->n_elems;
  if (op->host_conn.size() != size_t(E) * npe || op->elem_order.size() != size_t(E))
    validation("assemble_bcsr: operator setup data released");
  // node -> sweep positions, each row in ascending caller element id (the reference's sum order)
  std::vector<int64_t> iptr(size_t(n) + 1, 0);
  for (int64_t i = 0; i < E * npe; ++i) ++iptr[op->host_conn[i] + 1];
  for (int32_t r = 0; r < n; ++r) iptr[r + 1] += iptr[r];
  std::vector<int32_t> ipos(iptr[n]);
  {
    std::vector<int64_t> cur(iptr.begin(), iptr.end() - 1);
    for (int64_t i = 0; i < E; ++i)
      for (int a = 0; a < npe; ++a) ipos[cur[op->host_conn[i * npe + a]]++] = static_cast<int32_t>(i);
    for (int32_t r = 0; r < n; ++r)
      std::sort(ipos.begin() + iptr[r], ipos.begin() + iptr[r + 1],
                [&](int32_t x, int32_t y) { return op->elem_order[x] < op->elem_order[y]; });
  }
  std::vector<int32_t> rp(size_t(n) + 1, 0), ci;
  {
    std::vector<int32_t> row;
    for (int32_t r = 0; r < n; ++r) {
      row.clear();
      for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k)
        for (int a = 0; a < npe; ++a) row.push_back(op->host_conn[size_t(ipos[k]) * npe + a]);
      std::sort(row.begin(), row.end());
      row.erase(std::unique(row.begin(), row.end()), row.end());
      rp[r + 1] = rp[r] + static_cast<int32_t>(row.size());
      ci.insert(ci.end(), row.begin(), row.end());
    }
  }
  *nnzb = rp[n];
  if (!row_ptr && !col_idx && !blocks) return TS_OK;
  if (!row_ptr || !col_idx || !blocks) validation("assemble_bcsr: null argument");
  if (op->coef64.size() != 12 * size_t(E))
    validation("assemble_bcsr: operator setup data released (level-set inner operators keep only device state)");
  tsg::DevBuf<int64_t> d_iptr;
  tsg::DevBuf<int32_t> d_ipos, d_conn, d_rp, d_ci;
  tsg::DevBuf<double> d_c64, acc(9 * size_t(rp[n]));
  d_iptr.upload(iptr);
  d_ipos.upload(ipos);
  d_conn.upload(op->host_conn.data(), op->host_conn.size());
  d_c64.upload(op->coef64.data(), op->coef64.size());
  d_rp.upload(rp);
  d_ci.upload(ci);
  TS_CUDA(cudaMemset(acc.get(), 0, acc.size() * sizeof(double)));
  const uint8_t* mask = op->has_mask ? op->mask.get() : nullptr;
  if (n > 0) {
    if (npe == 10)
      tsg::k_assemble_rows<10><<<tsg::grid_for(n, 64), 64>>>(d_iptr.get(), d_ipos.get(), d_conn.get(), d_c64.get(),
                                                              mask, d_rp.get(), d_ci.get(), n, acc.get());
    else
      tsg::k_assemble_rows<4><<<tsg::grid_for(n, 64), 64>>>(d_iptr.get(), d_ipos.get(), d_conn.get(), d_c64.get(),
                                                             mask, d_rp.get(), d_ci.get(), n, acc.get());
    TS_CUDA_LAUNCH();
  }
  const int64_t len = 9 * int64_t(rp[n]);
  tsg::DevBuf<unsigned char> out(size_t(len) * tsg::tsize(op->prec));
  if (len > 0) {
    if (op->prec == 32)
      tsg::k_cast_blocks<float><<<tsg::grid_for(len, 256), 256>>>(acc.get(), reinterpret_cast<float*>(out.get()), len);
    else
      tsg::k_cast_blocks<double><<<tsg::grid_for(len, 256), 256>>>(acc.get(), reinterpret_cast<double*>(out.get()),
                                                                   len);
    TS_CUDA_LAUNCH();
  }
  std::memcpy(row_ptr, rp.data(), rp.size() * sizeof(int32_t));
  std::memcpy(col_idx, ci.data(), ci.size() * sizeof(int32_t));
  tsg::down(blocks, out.get(), size_t(len) * tsg::tsize(op->prec));
  TS_API_END
}

// ------------------------------------------------------------ level-2 setup (host, order-exact)
namespace {
tsg::BcsrD bcsr_from(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* blocks) {
  tsg::BcsrD a;
  a.n = n;
  a.row_ptr.assign(row_ptr, row_ptr + n + 1);
  a.col_idx.assign(col_idx, col_idx + row_ptr[n]);
  if (blocks) a.blocks.assign(blocks, blocks + 9 * size_t(row_ptr[n]));
  return a;
}
}  // namespace

// aggregate_p1 (aggregation.hpp:23-89): agg_of_node [n], seeds [n] (first *n_aggregates used)
ts_status ts_aggregate_p1(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, int32_t target,
                          int32_t* agg_of_node, int32_t* n_aggregates, int32_t* seeds) {
  TS_API_BEGIN
  if (!row_ptr || (n > 0 && (!col_idx || !agg_of_node)) || !n_aggregates) validation("aggregate_p1: null argument");
  const tsg::Aggregation agg = tsg::aggregate_p1(bcsr_from(n, row_ptr, col_idx, nullptr), target);
  std::memcpy(agg_of_node, agg.agg_of_node.data(), agg.agg_of_node.size() * sizeof(int32_t));
  *n_aggregates = agg.n_aggregates;
  if (seeds) std::memcpy(seeds, agg.seeds.data(), agg.seeds.size() * sizeof(int32_t));
  TS_API_END
}

// build_level2 (aggregation.hpp:95-170): the Galerkin A2 = P^T K1 P of an fp64 block-CSR K1
// (fine_mask [3 n] or NULL); NULL outputs -> *nnzb2 only
ts_status ts_build_level2(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* blocks,
                          const int32_t* agg_of_node, int32_t n_aggregates, const uint8_t* fine_mask, int64_t* nnzb2,
                          int32_t* row_ptr2, int32_t* col_idx2, double* blocks2) {
  TS_API_BEGIN
  if (!row_ptr || !nnzb2 || (n > 0 && (!col_idx || !blocks || !agg_of_node))) validation("build_level2: null argument");
  if (n_aggregates < 1) validation("build_level2: empty aggregation");
  std::vector<int32_t> count(n_aggregates, 0);
  for (int32_t r = 0; r < n; ++r) {
    const int32_t v = agg_of_node[r];
    if (v < 0 || v >= n_aggregates) validation("build_level2: node without aggregate");
    ++count[v];
  }
  for (int32_t c : count)
    if (c == 0) validation("build_level2: empty aggregate");
  tsg::Aggregation agg;
  agg.agg_of_node.assign(agg_of_node, agg_of_node + n);
  agg.n_aggregates = n_aggregates;
  std::vector<uint8_t> mask;
  if (fine_mask) mask.assign(fine_mask, fine_mask + 3 * size_t(n));
  const tsg::BcsrD a2 = tsg::build_level2(bcsr_from(n, row_ptr, col_idx, blocks), agg, mask);
  *nnzb2 = a2.row_ptr[a2.n];
  if (!row_ptr2 && !col_idx2 && !blocks2) return TS_OK;
  if (!row_ptr2 || !col_idx2 || !blocks2) validation("build_level2: null argument");
  std::memcpy(row_ptr2, a2.row_ptr.data(), a2.row_ptr.size() * sizeof(int32_t));
  std::memcpy(col_idx2, a2.col_idx.data(), a2.col_idx.size() * sizeof(int32_t));
  std::memcpy(blocks2, a2.blocks.data(), a2.blocks.size() * sizeof(double));
  TS_API_END
}

// ------------------------------------------------------------ column ops (host buffers)
ts_status ts_dot_columns_host(int32_t prec, int64_t ndof, int32_t batch, const void* x, const void* y, double* out) {
  TS_API_BEGIN
  tsg::check_prec(prec, "dot_columns");
  if (!x || !y || !out || batch < 1 || ndof < 0) validation("dot_columns: bad argument");
  tsg::require_device();
  const size_t bytes = size_t(ndof) * batch * tsg::tsize(prec);
  tsg::Staged st;
  const void* dx = st.in(x, bytes);
  const void* dy = st.in(y, bytes);
  tsg::DevBuf<double> d(batch);
  if (prec == 32)
    tsg::k_dot_columns<float><<<batch, 256>>>(static_cast<const float*>(dx), static_cast<const float*>(dy), ndof, batch,
                                              d.get());
  else
    tsg::k_dot_columns<double><<<batch, 256>>>(static_cast<const double*>(dx), static_cast<const double*>(dy), ndof,
                                               batch, d.get());
  TS_CUDA_LAUNCH();
  tsg::down(out, d.get(), batch * sizeof(double));
  TS_API_END
}

ts_status ts_axpy_columns_host(int32_t prec, int64_t ndof, int32_t batch, const double* alpha, const void* x,
                               void* y) {
  TS_API_BEGIN
  tsg::check_prec(prec, "axpy_columns");
  if (!alpha || !x || !y || batch < 1 || ndof < 0) validation("axpy_columns: bad argument");
  tsg::require_device();
  const int64_t len = ndof * batch;
  const size_t bytes = size_t(len) * tsg::tsize(prec);
  tsg::Staged st;
  const double* da = static_cast<const double*>(st.in(alpha, batch * sizeof(double)));
  const void* dx = st.in(x, bytes);
  void* dy = st.in(y, bytes);
  if (len > 0) {
    if (prec == 32)
      tsg::k_axpy_columns<float><<<tsg::grid_for(len, 256), 256>>>(da, static_cast<const float*>(dx),
                                                                   static_cast<float*>(dy), len, batch);
    else
      tsg::k_axpy_columns<double><<<tsg::grid_for(len, 256), 256>>>(da, static_cast<const double*>(dx),
                                                                    static_cast<double*>(dy), len, batch);
    TS_CUDA_LAUNCH();
  }
  tsg::down(y, dy, bytes);
  TS_API_END
}

ts_status ts_xpby_columns_host(int32_t prec, int64_t ndof, int32_t batch, const void* z, const double* beta,
                               void* p) {
  TS_API_BEGIN
  tsg::check_prec(prec, "xpby_columns");
  if (!beta || !z || !p || batch < 1 || ndof < 0) validation("xpby_columns: bad argument");
  tsg::require_device();
  const int64_t len = ndof * batch;
  const size_t bytes = size_t(len) * tsg::tsize(prec);
  tsg::Staged st;
  const void* dz = st.in(z, bytes);
  const double* db = static_cast<const double*>(st.in(beta, batch * sizeof(double)));
  void* dp = st.in(p, bytes);
  if (len > 0) {
    if (prec == 32)
      tsg::k_xpby_columns<float><<<tsg::grid_for(len, 256), 256>>>(static_cast<const float*>(dz), db,
                                                                   static_cast<float*>(dp), len, batch);
    else
      tsg::k_xpby_columns<double><<<tsg::grid_for(len, 256), 256>>>(static_cast<const double*>(dz), db,
                                                                    static_cast<double*>(dp), len, batch);
    TS_CUDA_LAUNCH();
  }
  tsg::down(p, dp, bytes);
  TS_API_END
}

ts_status ts_sub_columns_host(int32_t prec, int64_t n, const void* a, const void* b, void* out) {
  TS_API_BEGIN
  tsg::check_prec(prec, "sub_columns");
  if (!a || !b || !out || n < 0) validation("sub_columns: bad argument");
  tsg::require_device();
  const size_t bytes = size_t(n) * tsg::tsize(prec);
  tsg::Staged st;
  const void* da = st.in(a, bytes);
  const void* db = st.in(b, bytes);
  void* dout = st.out(bytes);
  if (n > 0) {
    if (prec == 32)
      tsg::k_sub_columns<float><<<tsg::grid_for(n, 256), 256>>>(static_cast<const float*>(da),
                                                                static_cast<const float*>(db),
                                                                static_cast<float*>(dout), n);
    else
      tsg::k_sub_columns<double><<<tsg::grid_for(n, 256), 256>>>(static_cast<const double*>(da),
                                                                 static_cast<const double*>(db),
                                                                 static_cast<double*>(dout), n);
    TS_CUDA_LAUNCH();
  }
  tsg::down(out, dout, bytes);
  TS_API_END
}

ts_status ts_zero_masked_host(int32_t prec, int64_t ndof, int32_t batch, void* x, const uint8_t* mask) {
  TS_API_BEGIN
  tsg::check_prec(prec, "zero_masked");
  if (!x || !mask || batch < 1 || ndof < 0) validation("zero_masked: bad argument");
  tsg::require_device();
  const int64_t len = ndof * batch;
  const size_t bytes = size_t(len) * tsg::tsize(prec);
  tsg::Staged st;
  void* dx = st.in(x, bytes);
  const uint8_t* dm = static_cast<const uint8_t*>(st.in(mask, size_t(ndof)));
  if (len > 0) {
    if (prec == 32)
      tsg::k_zero_masked<float><<<tsg::grid_for(len, 256), 256>>>(static_cast<float*>(dx), dm, len, batch);
    else
      tsg::k_zero_masked<double><<<tsg::grid_for(len, 256), 256>>>(static_cast<double*>(dx), dm, len, batch);
    TS_CUDA_LAUNCH();
  }
  tsg::down(x, dx, bytes);
  TS_API_END
}

ts_status ts_cast_batch_host(int32_t from_prec, int32_t to_prec, int64_t n, const void* x, void* y) {
  TS_API_BEGIN
  tsg::check_prec(from_prec, "cast_batch");
  tsg::check_prec(to_prec, "cast_batch");
  if (!x || !y || n < 0) validation("cast_batch: bad argument");
  tsg::require_device();
  tsg::Staged st;
  const void* dx = st.in(x, size_t(n) * tsg::tsize(from_prec));
  void* dy = st.out(size_t(n) * tsg::tsize(to_prec));
  if (n > 0) {
    const unsigned g = tsg::grid_for(n, 256);
    if (from_prec == 64 && to_prec == 32)
      tsg::k_cast<double, float><<<g, 256>>>(static_cast<const double*>(dx), static_cast<float*>(dy), n);
    else if (from_prec == 32 && to_prec == 64)
      tsg::k_cast<float, double><<<g, 256>>>(static_cast<const float*>(dx), static_cast<double*>(dy), n);
    else if (from_prec == 32)
      tsg::k_cast<float, float><<<g, 256>>>(static_cast<const float*>(dx), static_cast<float*>(dy), n);
    else
      tsg::k_cast<double, double><<<g, 256>>>(static_cast<const double*>(dx), static_cast<double*>(dy), n);
    TS_CUDA_LAUNCH();
  }
  tsg::down(y, dy, size_t(n) * tsg::tsize(to_prec));
  TS_API_END
}

}  // extern "C"
