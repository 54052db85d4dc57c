// blas.cu — the solve path's vector kernels: fused PCG/CG steps with
// deterministic per-column fp64 reductions, block Jacobi, level-2 BCSR,
// inter-grid transfers. Reference semantics cited per kernel.
//
// Reductions: every dot product accumulates in fp64 (vector_batch.hpp:51-64).
// A fixed grid (kRedBlocks) owns fixed entry ranges; each block writes one
// partial per column and a one-block finalize sums the partials in block
// order, so results are bit-reproducible run to run and column-independent
// (identical columns stay identical, test_solver.cpp:183-201).
#include <atomic>
#include <cfloat>
#include <stdexcept>
#include <cstdlib>
#include <cmath>

#include "blas.h"

namespace tsg {

namespace {

// W consecutive scalars (one 16 / 8-byte access), W | B so a pack never
// straddles two dof rows and its columns are b0 .. b0+W-1.
template <typename T, int W>
struct alignas(sizeof(T) * W) Pack {
  T v[W];
};
template <typename T, int W>
__device__ __forceinline__ Pack<T, W> ld(const T* p) {
  return *reinterpret_cast<const Pack<T, W>*>(p);
}
template <typename T, int W>
__device__ __forceinline__ void st(T* p, const Pack<T, W>& x) {
  *reinterpret_cast<Pack<T, W>*>(p) = x;
}

// Partial sums over a contiguous entry range per block. Each thread walks
// packs of W entries with a stride of S entries (S = largest multiple of B
// <= kRedThreads * W), so its columns b0..b0+W-1 never change; the block then
// sums each column's slots in fixed order, so results are reproducible and
// identical columns stay identical. `owned` (nullable, distributed solves):
// per-node flags; entries of nodes this rank does not own are visited
// (updates happen everywhere) but do not accumulate. Entry i belongs to node
// i / per_node. f(i0, b0, acc[ND][W], own) handles entries i0..i0+W-1.
template <int ND, int W, typename F>
__device__ __forceinline__ void reduce_pass(int64_t len, int32_t B, double* __restrict__ partial,
                                            const uint8_t* __restrict__ owned, int64_t per_node, F&& f) {
  __shared__ double sm[ND * kRedThreads * W];
  const int S = (kRedThreads * W / B) * B;
  const int t = threadIdx.x;
  double acc[ND][W];
#pragma unroll
  for (int k = 0; k < ND; ++k)
#pragma unroll
    for (int c = 0; c < W; ++c) acc[k][c] = 0.0;
  if (t * W < S) {
    const int b0 = (t * W) % B;
    const int64_t per = ((len + gridDim.x - 1) / gridDim.x + S - 1) / S * S;
    const int64_t lo = per * blockIdx.x;
    const int64_t hi = lo + per < len ? lo + per : len;
    if (owned) {
#pragma unroll 2
      for (int64_t i = lo + int64_t(t) * W; i < hi; i += S) f(i, b0, acc, owned[i / per_node] != 0);
    } else {
#pragma unroll 2
      for (int64_t i = lo + int64_t(t) * W; i < hi; i += S) f(i, b0, acc, true);
    }
  }
#pragma unroll
  for (int k = 0; k < ND; ++k)
#pragma unroll
    for (int c = 0; c < W; ++c) sm[k * kRedThreads * W + t * W + c] = acc[k][c];
  __syncthreads();
  if (t < B) {
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      double s = 0.0;
      for (int j = t; j < S; j += B) s += sm[k * kRedThreads * W + j];
      partial[(static_cast<int64_t>(blockIdx.x) * ND + k) * B + t] = s;
    }
  }
}

// Column totals of the nd x B partials over nblk blocks into shared memory,
// with every thread of the block: thread t sums the blocks t/P, t/P + T/P, ...
// of pair t % P (P = nd*B) in ascending order, then pair p's slots are added in
// slot order — a fixed order, so the totals are reproducible. tot[k*B + b].
__device__ void block_totals(const double* __restrict__ partial, int nd, int32_t B, int nblk,
                             double* __restrict__ tot, double* __restrict__ scratch) {
  const int P = nd * B, t = threadIdx.x;
  const int slots = blockDim.x / P;  // >= 1: P <= 4 * 256 and blockDim = 1024
  if (t < slots * P) {
    const int pr = t % P, s0 = t / P;
    double s = 0.0;
#pragma unroll 4
    for (int blk = s0; blk < nblk; blk += slots) s += partial[int64_t(blk) * P + pr];
    scratch[t] = s;
  }
  __syncthreads();
  if (t < P) {
    double s = 0.0;
    for (int j = 0; j < slots; ++j) s += scratch[j * P + t];
    tot[t] = s;
  }
  __syncthreads();
}
constexpr int kFinThreads = 1024;

// column total of partial k, read from block_totals' result
__device__ __forceinline__ double col_total(const double* __restrict__ tot, int k, int32_t B, int b) {
  return tot[k * B + b];
}

// max_rel_ratio (pcg.hpp:32-42): max_b num/den; 0/0 converged; x/0 -> inf
__device__ void write_ratio(const double* num, const double* den, int32_t B, PcgStatus* st) {
  if (threadIdx.x != 0) return;
  double worst = 0.0;
  bool inf = false;
  for (int b = 0; b < B; ++b) {
    if (den[b] == 0.0) {
      if (num[b] != 0.0) inf = true;
      continue;
    }
    const double q = num[b] / den[b];
    if (q > worst || isnan(q)) worst = isnan(q) ? q : (isnan(worst) ? worst : q);
  }
  const double r = inf ? INFINITY : worst;
  st->ratio = r;
  st->nonfinite = isnan(r) ? 1 : 0;
}

// ---------------------------------------------------------------- kernels
template <typename T, int W>
__global__ void __launch_bounds__(kRedThreads) k_dot2(const T* __restrict__ x0, const T* __restrict__ y0,
                                                      const T* __restrict__ x1, const T* __restrict__ y1,
                                                      int64_t len, int32_t B, double* partial,
                                                      const uint8_t* __restrict__ owned) {
  if (x1) {
    reduce_pass<2, W>(len, B, partial, owned, 3 * int64_t(B), [&](int64_t i, int, double(&acc)[2][W], bool own) {
      if (!own) return;
      const Pack<T, W> a = ld<T, W>(x0 + i), c = ld<T, W>(y0 + i), d = ld<T, W>(x1 + i), e = ld<T, W>(y1 + i);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        acc[0][k] += double(a.v[k]) * double(c.v[k]);
        acc[1][k] += double(d.v[k]) * double(e.v[k]);
      }
    });
  } else {
    reduce_pass<1, W>(len, B, partial, owned, 3 * int64_t(B), [&](int64_t i, int, double(&acc)[1][W], bool own) {
      if (!own) return;
      const Pack<T, W> a = ld<T, W>(x0 + i), c = ld<T, W>(y0 + i);
#pragma unroll
      for (int k = 0; k < W; ++k) acc[0][k] += double(a.v[k]) * double(c.v[k]);
    });
  }
}

__global__ void __launch_bounds__(kFinThreads) k_sum_partials(const double* partial, int nd, int32_t B, int nblk,
                                                              double* out) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  block_totals(partial, nd, B, nblk, tot, scr);
  const int t = threadIdx.x;
  if (t < nd * B) out[t] = tot[t];
}

// z = M^-1 e per node (fp64 math, rounded to T); entries are (node, case)
template <typename T, int W>
__device__ __forceinline__ void bj_pack(const T* __restrict__ m, const Pack<T, W> (&ev)[3], Pack<T, W> (&z)[3]) {
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const double e0 = double(ev[0].v[k]), e1 = double(ev[1].v[k]), e2 = double(ev[2].v[k]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      z[i].v[k] = static_cast<T>(double(m[3 * i]) * e0 + double(m[3 * i + 1]) * e1 + double(m[3 * i + 2]) * e2);
  }
}

// accumulate (M^-1 e, e)
template <typename T, int W>
__global__ void __launch_bounds__(kRedThreads) k_rho(const T* __restrict__ inv, const T* __restrict__ e,
                                                     int32_t n, int32_t B, double* partial,
                                                     const uint8_t* __restrict__ owned) {
  reduce_pass<1, W>(int64_t(n) * B, B, partial, owned, int64_t(B), [&](int64_t it, int b0, double(&acc)[1][W], bool own) {
    if (!own) return;
    const int64_t node = it / B;
    const T* ev = e + 3 * node * B + b0;
    const Pack<T, W> x[3] = {ld<T, W>(ev), ld<T, W>(ev + B), ld<T, W>(ev + 2 * B)};
    Pack<T, W> z[3];
    bj_pack<T, W>(inv + 9 * node, x, z);
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int i = 0; i < 3; ++i) acc[0][k] += double(z[i].v[k]) * double(x[i].v[k]);
  });
}

__global__ void __launch_bounds__(kFinThreads) k_rho_final(const double* partial, int nd, int slot, int nblk,
                                                           int32_t B, int first, double* rho_a, const double* rho_b,
                                                           double* beta) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  block_totals(partial, nd, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b >= B) return;
  const double r = tot[slot * B + b];
  rho_a[b] = r;
  beta[b] = first ? 0.0 : (rho_b[b] != 0.0 ? r / rho_b[b] : 0.0);  // pcg.hpp:74-80
}

// p = z + (T)beta p, z = M^-1 e (xpby_columns, vector_batch.hpp:86-97); first: p = z.
// q (optional): the next EBE product's starting value, the masked identity of
// the new p (ebe_operator.hpp:96-110), written here so the product skips its own
// initialisation pass (mask null: zeros).
// u (optional): the previous iteration's u += (T)alpha p (pcg.hpp:112-113), applied
// here, where the old p is read anyway, instead of in the update pass — the same
// operation on the same values, one vector read fewer per iteration.
template <typename T, int W>
__global__ void k_direction(const T* __restrict__ inv, const T* __restrict__ e, T* __restrict__ p, int32_t n,
                            int32_t B, int first, const double* __restrict__ beta, T* __restrict__ q,
                            const uint8_t* __restrict__ mask, T* __restrict__ u, const double* __restrict__ alpha) {
  const int64_t it = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * W;
  if (it >= int64_t(n) * B) return;
  const int64_t node = it / B;
  const int b0 = static_cast<int>(it - node * B);
  const T* ev = e + 3 * node * B + b0;
  T* pv = p + 3 * node * B + b0;
  const Pack<T, W> x[3] = {ld<T, W>(ev), ld<T, W>(ev + B), ld<T, W>(ev + 2 * B)};
  Pack<T, W> z[3];
  bj_pack<T, W>(inv + 9 * node, x, z);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (!first) {
      const Pack<T, W> pp = ld<T, W>(pv + i * B);
#pragma unroll
      for (int k = 0; k < W; ++k) z[i].v[k] = z[i].v[k] + static_cast<T>(beta[b0 + k]) * pp.v[k];
      if (u) {
        T* uv = u + 3 * node * B + b0 + i * B;
        Pack<T, W> x = ld<T, W>(uv);
#pragma unroll
        for (int k = 0; k < W; ++k) x.v[k] = x.v[k] + static_cast<T>(alpha[b0 + k]) * pp.v[k];
        st<T, W>(uv, x);
      }
    }
    st<T, W>(pv + i * B, z[i]);
    if (q) {
      Pack<T, W> qi;
      const bool keep = mask && mask[3 * node + i];
#pragma unroll
      for (int k = 0; k < W; ++k) qi.v[k] = keep ? z[i].v[k] : T(0);
      st<T, W>(q + 3 * node * B + b0 + i * B, qi);
    }
  }
}

template <typename T, int W>
__global__ void __launch_bounds__(kRedThreads) k_gamma(const T* __restrict__ p, const T* __restrict__ q, int64_t len,
                                                       int32_t B, double* partial, const uint8_t* __restrict__ owned) {
  reduce_pass<3, W>(len, B, partial, owned, 3 * int64_t(B), [&](int64_t i, int, double(&acc)[3][W], bool own) {
    if (!own) return;
    const Pack<T, W> a = ld<T, W>(p + i), c = ld<T, W>(q + i);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const double x = double(a.v[k]), y = double(c.v[k]);
      acc[0][k] += x * y;
      acc[1][k] += x * x;
      acc[2][k] += y * y;
    }
  });
}

// alpha with the reference's breakdown / stagnation rules (pcg.hpp:83-110)
template <typename T>
__global__ void __launch_bounds__(kFinThreads) k_gamma_final(const double* partial, int nblk, int32_t B,
                                                             const double* rho_a, double* rho_b, double* gamma,
                                                             double* alpha, PcgStatus* st, int pq_only = 0) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  __shared__ int stag, brk, full;
  if (threadIdx.x == 0) {
    stag = 0;
    brk = INT32_MAX;
    full = 0;
  }
  block_totals(partial, 3, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b < B) {
    const double g = tot[b];
    gamma[b] = g;
    double a = 0.0;
    if (pq_only > 1) {  // test hook (TSGPU_TEST_FUSED_FALLBACK): every iteration takes the full-pass fallback
      atomicExch(&full, 1);
    } else if (g > 0.0) {
      a = rho_a[b] / g;
    } else if (g == 0.0 && rho_a[b] == 0.0) {
      a = 0.0;
    } else if (pq_only) {
      atomicExch(&full, 1);  // ||p||, ||q|| unknown here: the full pass decides
      a = 0.0;
    } else {
      const double pn = tot[B + b], qn = tot[2 * B + b];
      const double scale = sqrt(pn) * sqrt(qn);
      const double eps16 = 16.0 * (sizeof(T) == 4 ? double(FLT_EPSILON) : DBL_EPSILON);
      if (fabs(g) <= eps16 * scale) atomicExch(&stag, 1);
      else atomicMin(&brk, b);
      a = 0.0;
    }
    alpha[b] = a;
  }
  __syncthreads();
  if (b < B && !stag && brk == INT32_MAX && !full) rho_b[b] = rho_a[b];
  if (threadIdx.x == 0) {
    st->stagnated = stag;
    st->breakdown_col = brk == INT32_MAX ? -1 : brk;
    st->need_full = full;
  }
}

// e += (T)(-alpha) q (axpy_columns, vector_batch.hpp:72-83); partials ||e||^2 and
// — for the next iteration's beta — (M^-1 e, e) (pcg.hpp:72-73,116), one pass over
// the node's 3 dofs x W cases. u += (T)alpha p is deferred to the next direction
// pass (or pcg_apply_pending when the loop ends).
template <typename T, int W>
__global__ void __launch_bounds__(kRedThreads) k_update(const T* __restrict__ inv, T* __restrict__ e,
                                                        const T* __restrict__ q, int32_t n, int32_t B,
                                                        const double* __restrict__ alpha,
                                                        const PcgStatus* __restrict__ st_, double* partial,
                                                        const uint8_t* __restrict__ owned) {
  const bool skip = st_->stagnated || st_->breakdown_col >= 0 || st_->need_full;
  reduce_pass<2, W>(int64_t(n) * B, B, partial, owned, int64_t(B), [&](int64_t it, int b0, double(&acc)[2][W], bool own) {
    const int64_t node = it / B;
    const int64_t base = 3 * node * B + b0;
    Pack<T, W> ev[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) ev[i] = ld<T, W>(e + base + i * B);
    if (!skip) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const Pack<T, W> qv = ld<T, W>(q + base + i * B);
#pragma unroll
        for (int k = 0; k < W; ++k) ev[i].v[k] = ev[i].v[k] + static_cast<T>(-alpha[b0 + k]) * qv.v[k];
        st<T, W>(e + base + i * B, ev[i]);
      }
    }
    if (!own) return;
    Pack<T, W> z[3];
    bj_pack<T, W>(inv + 9 * node, ev, z);
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        acc[0][k] += double(ev[i].v[k]) * double(ev[i].v[k]);
        acc[1][k] += double(z[i].v[k]) * double(ev[i].v[k]);
      }
  });
}

// u += (T)alpha p: the last iteration's deferred update (see k_direction)
template <typename T, int W>
__global__ void k_apply_pending(T* __restrict__ u, const T* __restrict__ p, int32_t n, int32_t B,
                                const double* __restrict__ alpha) {
  const int64_t it = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * W;
  if (it >= 3 * int64_t(n) * B) return;
  const int b0 = static_cast<int>(it % B);
  Pack<T, W> x = ld<T, W>(u + it);
  const Pack<T, W> pp = ld<T, W>(p + it);
#pragma unroll
  for (int k = 0; k < W; ++k) x.v[k] = x.v[k] + static_cast<T>(alpha[b0 + k]) * pp.v[k];
  st<T, W>(u + it, x);
}

__global__ void __launch_bounds__(kFinThreads) k_ratio_final(const double* partial, int nd, int nblk, int32_t B,
                                                             double* num, const double* den, PcgStatus* st) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  block_totals(partial, nd, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b < B) num[b] = tot[b];
  __syncthreads();
  write_ratio(num, den, B, st);
}

// e = r - e (e holds A u); partials ||r||^2, ||e||^2 (pcg.hpp:59-65) and (M^-1 e, e)
template <typename T, int W>
__global__ void __launch_bounds__(kRedThreads) k_init(const T* __restrict__ inv, const T* __restrict__ r,
                                                      T* __restrict__ e, int32_t n, int32_t B, double* partial,
                                                      const uint8_t* __restrict__ owned) {
  reduce_pass<3, W>(int64_t(n) * B, B, partial, owned, int64_t(B), [&](int64_t it, int b0, double(&acc)[3][W], bool own) {
    const int64_t node = it / B;
    const int64_t base = 3 * node * B + b0;
    Pack<T, W> rv[3], ev[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rv[i] = ld<T, W>(r + base + i * B);
      ev[i] = ld<T, W>(e + base + i * B);
#pragma unroll
      for (int k = 0; k < W; ++k) ev[i].v[k] = rv[i].v[k] - ev[i].v[k];
      st<T, W>(e + base + i * B, ev[i]);
    }
    if (!own) return;
    Pack<T, W> z[3];
    bj_pack<T, W>(inv + 9 * node, ev, z);
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        acc[0][k] += double(rv[i].v[k]) * double(rv[i].v[k]);
        acc[1][k] += double(ev[i].v[k]) * double(ev[i].v[k]);
        acc[2][k] += double(z[i].v[k]) * double(ev[i].v[k]);
      }
  });
}

__global__ void __launch_bounds__(kFinThreads) k_init_final(const double* partial, int nblk, int32_t B, double* rn2,
                                                            double* en2, PcgStatus* st) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  block_totals(partial, 3, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b < B) {
    rn2[b] = tot[b];
    en2[b] = tot[B + b];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->stagnated = 0;
    st->breakdown_col = -1;
    st->need_full = 0;
  }
  write_ratio(en2, rn2, B, st);
}

// ---- outer CG (fp64) ----
template <int W>
__global__ void __launch_bounds__(kRedThreads) k_true_res(const double* __restrict__ f, double* __restrict__ r,
                                                          int64_t len, int32_t B, double* partial,
                                                          const uint8_t* __restrict__ owned) {
  reduce_pass<1, W>(len, B, partial, owned, 3 * int64_t(B), [&](int64_t i, int, double(&acc)[1][W], bool own) {
    const Pack<double, W> fv = ld<double, W>(f + i);
    Pack<double, W> rv = ld<double, W>(r + i);
#pragma unroll
    for (int k = 0; k < W; ++k) rv.v[k] = fv.v[k] - rv.v[k];
    st<double, W>(r + i, rv);
    if (own)
#pragma unroll
      for (int k = 0; k < W; ++k) acc[0][k] += rv.v[k] * rv.v[k];
  });
}

__global__ void __launch_bounds__(kFinThreads) k_cg_beta(const double* partial, int nblk, int32_t B,
                                                         const double* gprev, double* beta) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  block_totals(partial, 1, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b >= B) return;
  const double zq = tot[b];
  beta[b] = gprev[b] != 0.0 ? -zq / gprev[b] : 0.0;  // adaptive_cg.hpp:196-200
}

__global__ void k_xpby(const double* __restrict__ z, double* __restrict__ p, int64_t len, int32_t B, int first,
                       const double* __restrict__ beta) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= len) return;
  p[i] = first ? z[i] : z[i] + beta[i % B] * p[i];
}

__global__ void __launch_bounds__(kFinThreads) k_cg_alpha(const double* partial, int nblk, int32_t B, double* rho,
                                                          double* gamma, double* gprev, double* alpha, PcgStatus* st) {
  __shared__ double tot[kFinThreads], scr[kFinThreads];
  __shared__ int brk;
  if (threadIdx.x == 0) brk = INT32_MAX;
  block_totals(partial, 2, B, nblk, tot, scr);
  const int b = threadIdx.x;
  if (b < B) {
    const double r = tot[b], g = tot[B + b];
    rho[b] = r;
    gamma[b] = g;
    double a = 0.0;
    if (g > 0.0) a = r / g;
    else if (g == 0.0 && r == 0.0) a = 0.0;
    else atomicMin(&brk, b);  // adaptive_cg.hpp:205-213
    alpha[b] = a;
    gprev[b] = g;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->stagnated = 0;
    st->breakdown_col = brk == INT32_MAX ? -1 : brk;
    st->need_full = 0;
  }
}

template <int W>
__global__ void __launch_bounds__(kRedThreads) k_cg_update(double* __restrict__ r, double* __restrict__ u,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ q, int64_t len, int32_t B,
                                                           const double* __restrict__ alpha, double* partial,
                                                           const uint8_t* __restrict__ owned) {
  reduce_pass<1, W>(len, B, partial, owned, 3 * int64_t(B), [&](int64_t i, int b0, double(&acc)[1][W], bool own) {
    Pack<double, W> rv = ld<double, W>(r + i), uv = ld<double, W>(u + i);
    const Pack<double, W> pv = ld<double, W>(p + i), qv = ld<double, W>(q + i);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const double a = alpha[b0 + k];
      rv.v[k] = rv.v[k] + (-a) * qv.v[k];
      uv.v[k] = uv.v[k] + a * pv.v[k];
    }
    st<double, W>(r + i, rv);
    st<double, W>(u + i, uv);
    if (own)
#pragma unroll
      for (int k = 0; k < W; ++k) acc[0][k] += rv.v[k] * rv.v[k];
  });
}

// ---- small operators ----
template <typename T>
__global__ void k_bj_apply(const T* __restrict__ inv, const T* __restrict__ r, T* __restrict__ z, int32_t n,
                           int32_t B) {
  const int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (it >= int64_t(n) * B) return;
  const int64_t node = it / B;
  const int b = static_cast<int>(it % B);
  const T* m = inv + 9 * node;
  const T* rv = r + 3 * node * B + b;
  const double r0 = double(rv[0]), r1 = double(rv[B]), r2 = double(rv[2 * B]);
  T* zv = z + 3 * node * B + b;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    zv[i * B] = static_cast<T>(double(m[3 * i]) * r0 + double(m[3 * i + 1]) * r1 + double(m[3 * i + 2]) * r2);
}

// one thread per (block row, case): 3 outputs, fp64 accumulation in the
// reference's order a[b] += b0 u0 + b1 u1 + b2 u2 per stored block
__global__ void k_bcsr(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                       const float* __restrict__ blocks, int32_t n, const float* __restrict__ u,
                       float* __restrict__ f, int32_t B) {
  const int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (it >= int64_t(n) * B) return;
  const int32_t r = static_cast<int32_t>(it / B);
  const int b = static_cast<int>(it % B);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int32_t e = __ldg(row_ptr + r); e < __ldg(row_ptr + r + 1); ++e) {
    const float* blk = blocks + 9 * int64_t(e);
    const float* uc = u + 3 * int64_t(__ldg(col_idx + e)) * B + b;
    const double u0 = double(uc[0]), u1 = double(uc[B]), u2 = double(uc[2 * B]);
    a0 += double(blk[0]) * u0 + double(blk[1]) * u1 + double(blk[2]) * u2;
    a1 += double(blk[3]) * u0 + double(blk[4]) * u1 + double(blk[5]) * u2;
    a2 += double(blk[6]) * u0 + double(blk[7]) * u1 + double(blk[8]) * u2;
  }
  float* fr = f + 3 * int64_t(r) * B + b;
  fr[0] = static_cast<float>(a0);
  fr[B] = static_cast<float>(a1);
  fr[2 * B] = static_cast<float>(a2);
}

// Assembled level-1 operator (K1 of the fp32 tier, setup.cpp assemble_tet4):
// W cases of one block row per thread, fp32 accumulation of ~14 blocks — the
// EbeOperator<float> order-1 product (fp32 cross-element sums) without atomics.
// ACC = float: the level-1 operator (fp32 sums); ACC = double: level 2 with the
// reference's fp64 row accumulation in stored-block order (block_csr.hpp:40-54)
template <int W, typename ACC>
__global__ void k_bcsr_rows(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                            const float* __restrict__ blocks, int32_t n, const float* __restrict__ u,
                            float* __restrict__ f, int32_t B, const int32_t* __restrict__ rows) {
  const int qpr = B / W;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t k = t / qpr;
  if (k >= n) return;
  const int b0 = static_cast<int>(t - k * qpr) * W;
  const int64_t r = rows ? int64_t(__ldg(rows + k)) : k;  // rows (nullable): a subset of the rows, in this order
  ACC acc[3][W];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < W; ++k) acc[i][k] = ACC(0);
  const int32_t e1 = __ldg(row_ptr + r + 1);
  // unrolled so the loads of several blocks (index -> u gathers) are in flight together
#pragma unroll 4
  for (int32_t e = __ldg(row_ptr + r); e < e1; ++e) {
    const float* blk = blocks + 9 * int64_t(e);
    float m[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) m[q] = __ldg(blk + q);
    const float* uc = u + 3 * int64_t(__ldg(col_idx + e)) * B + b0;
    const Pack<float, W> x0 = ld<float, W>(uc), x1 = ld<float, W>(uc + B), x2 = ld<float, W>(uc + 2 * B);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if constexpr (sizeof(ACC) == 4)
          acc[i][k] = fmaf(m[3 * i + 2], x2.v[k], fmaf(m[3 * i + 1], x1.v[k], fmaf(m[3 * i], x0.v[k], acc[i][k])));
        else  // a[b] += b0 u0 + b1 u1 + b2 u2 (block_csr.hpp:50)
          acc[i][k] += double(m[3 * i]) * double(x0.v[k]) + double(m[3 * i + 1]) * double(x1.v[k]) +
                       double(m[3 * i + 2]) * double(x2.v[k]);
      }
  }
  float* fr = f + 3 * r * B + b0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    Pack<float, W> o;
#pragma unroll
    for (int k = 0; k < W; ++k) o.v[k] = static_cast<float>(acc[i][k]);
    st<float, W>(fr + i * B, o);
  }
}

// The level-1 product with each warp's block rows staged in shared memory: a warp owns RPW
// consecutive rows (qpr = B / W threads each); their blocks and column indices are one
// contiguous range of the BCSR arrays, brought in by two bulk copies (TMA, completing on a
// per-warp mbarrier) instead of nine scalar loads per block and thread (which held k_bcsr_rows
// at the L1 request limit). Same sums in the same order as k_bcsr_rows. A warp whose range
// exceeds the staging capacity (or would read past the arrays' ends) loads from global memory.
constexpr int kStageWarps = 8;
template <int RPW, int PER_ROW = 20>
struct StageCap {
  static constexpr int kBlocks = RPW * PER_ROW + 8;                         // blocks per warp
  static constexpr int kBlkBytes = (kBlocks * 36 + 16 + 15) & ~15;         // + alignment slack
  static constexpr int kColBytes = (kBlocks * 4 + 16 + 15) & ~15;
  static constexpr int kWarpBytes = kBlkBytes + kColBytes + 16;             // + mbarrier
  static_assert(kBlkBytes % 16 == 0 && kColBytes % 16 == 0, "16-byte aligned staging regions");
};

// DOTS: a persistent grid (each warp strides over row sets) that also accumulates, per column, the
// fp64 dots (p, q), (p, p), (q, q) of the product's input p and output q over its rows — the inner
// PCG's gamma pass (k_gamma, pcg.hpp:82-88) without re-reading p and q — into per-block partials in
// the reduce_pass layout, in a fixed order (static row-set assignment; shuffles, then warps in order).
template <int W, int RPW, typename ACC, int PER_ROW = 20, bool DOTS = false>
__global__ void __launch_bounds__(32 * kStageWarps)
k_bcsr_rows_staged(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                   const float* __restrict__ blocks, int32_t n, int64_t nnz, const float* __restrict__ u,
                   float* __restrict__ f, int32_t B, double* __restrict__ partial,
                   const uint8_t* __restrict__ rowsel) {
  using Cap = StageCap<RPW, PER_ROW>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double red[DOTS ? kStageWarps * 3 * 32 : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int qpr = 32 / RPW;
  unsigned char* const wb = smem + size_t(wid) * Cap::kWarpBytes;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(wb + Cap::kBlkBytes + Cap::kColBytes);
  const unsigned sbar = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int b0 = (lane % qpr) * W;
  const float* ub = u + b0;
  unsigned phase = 0;
  double dacc[3][W];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int c = 0; c < W; ++c) dacc[k][c] = 0.0;
  const int64_t stride = int64_t(gridDim.x) * kStageWarps * RPW;
  for (int64_t r0 = (int64_t(blockIdx.x) * kStageWarps + wid) * RPW; r0 < n; r0 += stride) {
    const int64_t r1 = r0 + RPW < n ? r0 + RPW : n;
    const int64_t eb = __ldg(row_ptr + r0), ee = __ldg(row_ptr + r1);
    const int64_t bb0 = (eb * 36) & ~int64_t(15), bb1 = (ee * 36 + 15) & ~int64_t(15);
    const int64_t cb0 = (eb * 4) & ~int64_t(15), cb1 = (ee * 4 + 15) & ~int64_t(15);
    const bool staged = bb1 - bb0 <= Cap::kBlkBytes && cb1 - cb0 <= Cap::kColBytes && bb1 <= nnz * 36 &&
                        cb1 <= nnz * 4 && ee > eb;
    if (staged && lane == 0) {
      // the previous row set's shared reads (generic proxy) come before these async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar),
                   "r"(static_cast<unsigned>(bb1 - bb0 + cb1 - cb0))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(wb))),
                   "l"(reinterpret_cast<const unsigned char*>(blocks) + bb0), "r"(static_cast<unsigned>(bb1 - bb0)),
                   "r"(sbar)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(wb + Cap::kBlkBytes))),
                   "l"(reinterpret_cast<const unsigned char*>(col_idx) + cb0), "r"(static_cast<unsigned>(cb1 - cb0)),
                   "r"(sbar)
                   : "memory");
    }
    const int64_t r = r0 + lane / qpr;
    ACC acc[3][W];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int c = 0; c < W; ++c) acc[i][c] = ACC(0);
    const bool live = r < r1;
    const int32_t e0 = live ? __ldg(row_ptr + r) : 0, e1 = live ? __ldg(row_ptr + r + 1) : 0;
    auto block_step = [&](const float (&m)[9], int32_t col) {
      const float* uc = ub + 3 * int64_t(col) * B;
      const Pack<float, W> x0 = ld<float, W>(uc), x1 = ld<float, W>(uc + B), x2 = ld<float, W>(uc + 2 * B);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < W; ++c) {
          if constexpr (sizeof(ACC) == 4)
            acc[i][c] = fmaf(m[3 * i + 2], x2.v[c], fmaf(m[3 * i + 1], x1.v[c], fmaf(m[3 * i], x0.v[c], acc[i][c])));
          else
            acc[i][c] += double(m[3 * i]) * double(x0.v[c]) + double(m[3 * i + 1]) * double(x1.v[c]) +
                         double(m[3 * i + 2]) * double(x2.v[c]);
        }
    };
    if (staged) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(done)
                     : "r"(sbar), "r"(phase)
                     : "memory");
      phase ^= 1u;
      const unsigned char* const sb = wb - bb0;                 // byte address of block entry e: sb + 36 e
      const int32_t* const sc = reinterpret_cast<const int32_t*>(wb + Cap::kBlkBytes - cb0);  // sc[e]
#pragma unroll 4
      for (int32_t e = e0; e < e1; ++e) {
        const float* blk = reinterpret_cast<const float*>(sb + 36 * int64_t(e));
        float m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = blk[q];
        block_step(m, sc[e]);
      }
    } else {
#pragma unroll 4
      for (int32_t e = e0; e < e1; ++e) {
        const float* blk = blocks + 9 * int64_t(e);
        float m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = __ldg(blk + q);
        block_step(m, __ldg(col_idx + e));
      }
    }
    if (live) {
      float* fr = f + 3 * r * B + b0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        Pack<float, W> o;
#pragma unroll
        for (int c = 0; c < W; ++c) o.v[c] = static_cast<float>(acc[i][c]);
        st<float, W>(fr + i * B, o);
        if constexpr (DOTS) {
          if (rowsel && !rowsel[r]) continue;  // (partitioned: other ranks' rows / rows completed later)
          const Pack<float, W> pv = ld<float, W>(u + 3 * r * B + b0 + i * B);
#pragma unroll
          for (int c = 0; c < W; ++c) {
            const double x = double(pv.v[c]), y = double(o.v[c]);
            dacc[0][c] += x * y;
            dacc[1][c] += x * x;
            dacc[2][c] += y * y;
          }
        }
      }
    }
    __syncwarp();  // every lane is done with this row set's staging before it is refilled
    if constexpr (!DOTS) break;
  }
  if constexpr (DOTS) {
    // lanes l, l + qpr, ... hold the same columns: fold them (fixed shuffle order), then the warps in order
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int c = 0; c < W; ++c) {
        double v = dacc[k][c];
        for (int off = qpr; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane < qpr) red[(wid * 3 + k) * 32 + b0 + c] = v;
      }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < 3 * B) {
      const int k = t / B, b = t - k * B;
      double sum = 0.0;
      for (int w = 0; w < kStageWarps; ++w) sum += red[(w * 3 + k) * 32 + b];
      partial[(int64_t(blockIdx.x) * 3 + k) * B + b] = sum;
    }
  }
}

template <int W, int RPW, typename ACC, int PER_ROW = 20, bool DOTS = false>
int launch_rows_staged(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n, int64_t nnz,
                       const float* u, float* f, int32_t B, cudaStream_t s, double* partial = nullptr,
                       const uint8_t* rowsel = nullptr) {
  const size_t smem = size_t(kStageWarps) * StageCap<RPW, PER_ROW>::kWarpBytes;
  auto kern = k_bcsr_rows_staged<W, RPW, ACC, PER_ROW, DOTS>;
  // the shared-memory opt-in is a per-device attribute of the function: set once per device
  constexpr int kMaxDevices = 64;
  static std::atomic<int> per_sm[kMaxDevices] = {};  // 0: not configured yet
  static std::atomic<int> sms[kMaxDevices] = {};
  int dev = 0;
  TS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("bcsr rows: device ordinal out of range");
  if (per_sm[dev].load(std::memory_order_acquire) == 0) {
    TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int ps = 0, ns = 0;
    TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, 32 * kStageWarps, smem));
    TS_CUDA(cudaDeviceGetAttribute(&ns, cudaDevAttrMultiProcessorCount, dev));
    sms[dev].store(ns, std::memory_order_relaxed);
    per_sm[dev].store(std::max(ps, 1), std::memory_order_release);
  }
  static const bool force_global = [] {  // test hook: every warp takes the unstaged (global-load) path
    const char* e = std::getenv("TSGPU_STAGE_FORCE_GLOBAL");
    return e && e[0] == '1';
  }();
  if (force_global) nnz = 0;
  const int64_t rows_per_block = int64_t(kStageWarps) * RPW;
  int64_t grid = (n + rows_per_block - 1) / rows_per_block;
  if (DOTS)  // persistent: one resident wave (the partial count the finalize sums), at most kRedBlocks
    grid = std::min<int64_t>(grid, std::min<int64_t>(kRedBlocks, int64_t(sms[dev].load()) * per_sm[dev].load()));
  kern<<<static_cast<unsigned>(grid), 32 * kStageWarps, smem, s>>>(row_ptr, col_idx, blocks, n, nnz, u, f, B,
                                                                   partial, rowsel);
  return static_cast<int>(grid);
}

__global__ void k_cast_d2f(const double* __restrict__ x, float* __restrict__ y, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = static_cast<float>(x[i]);
}
__global__ void k_cast_f2d(const float* __restrict__ x, double* __restrict__ y, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = static_cast<double>(x[i]);
}
__global__ void k_zero_masked(float* __restrict__ x, const uint8_t* __restrict__ mask, int64_t len, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len && mask[i / B]) x[i] = 0.0f;
}

// out = 0 ; out += w * in per stored entry (float ops, no contraction)
__global__ void k_p1_apply(const float* __restrict__ c, float* __restrict__ fine, const int32_t* __restrict__ ends,
                           int32_t nv, int32_t nf, const uint8_t* __restrict__ mask, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = 3 * int64_t(nf) * B;
  if (i >= len) return;
  const int64_t dof = i / B;
  const int64_t node = dof / 3;
  const int64_t rem = i - node * 3 * B;  // axis * B + b
  float v;
  if (node < nv) {
    v = c[i];
  } else {
    const int64_t k = node - nv;
    const float a = c[3 * int64_t(ends[2 * k]) * B + rem];
    const float bb = c[3 * int64_t(ends[2 * k + 1]) * B + rem];
    v = __fadd_rn(__fmul_rn(0.5f, a), __fmul_rn(0.5f, bb));
  }
  fine[i] = (mask && mask[dof]) ? 0.0f : v;
}

__global__ void k_p1_restrict(const float* __restrict__ fine, float* __restrict__ coarse,
                              const int32_t* __restrict__ t_ptr, const int32_t* __restrict__ t_idx, int32_t nv,
                              const uint8_t* __restrict__ mask, int32_t B, const uint8_t* __restrict__ owned) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = 3 * int64_t(nv) * B;
  if (i >= len) return;
  const int64_t dof = i / B;
  const int64_t node = dof / 3;
  const int64_t rem = i - node * 3 * B;
  // fn = node itself first (weight 1); a partition adds it only on the owner
  float v = (owned && !owned[node]) ? 0.0f : 0.0f + fine[i];
  for (int32_t k = t_ptr[node]; k < t_ptr[node + 1]; ++k)
    v = __fadd_rn(v, __fmul_rn(0.5f, fine[3 * int64_t(t_idx[k]) * B + rem]));
  coarse[i] = (mask && mask[dof]) ? 0.0f : v;
}

__global__ void k_p2_apply(const float* __restrict__ c, float* __restrict__ fine, const int32_t* __restrict__ agg,
                           int32_t nf, const uint8_t* __restrict__ mask, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = 3 * int64_t(nf) * B;
  if (i >= len) return;
  const int64_t dof = i / B;
  const int64_t node = dof / 3;
  const int64_t rem = i - node * 3 * B;
  const float v = 0.0f + c[3 * int64_t(agg[node]) * B + rem];
  fine[i] = (mask && mask[dof]) ? 0.0f : v;
}

__global__ void k_p2_restrict(const float* __restrict__ fine, float* __restrict__ coarse,
                              const int32_t* __restrict__ a_ptr, const int32_t* __restrict__ a_idx, int32_t nc,
                              const uint8_t* __restrict__ mask, int32_t B) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t len = 3 * int64_t(nc) * B;
  if (i >= len) return;
  const int64_t dof = i / B;
  const int64_t node = dof / 3;
  const int64_t rem = i - node * 3 * B;
  float v = 0.0f;
  for (int32_t k = a_ptr[node]; k < a_ptr[node + 1]; ++k) v = __fadd_rn(v, fine[3 * int64_t(a_idx[k]) * B + rem]);
  coarse[i] = (mask && mask[dof]) ? 0.0f : v;
}

// pack width for batch B: 16-byte packs for fp32 (B % 4 == 0), else 8 / 4 bytes
template <typename T>
int pack_width(int32_t B) {
  if (sizeof(T) == 4) return B % 4 == 0 ? 4 : (B % 2 == 0 ? 2 : 1);
  return B % 2 == 0 ? 2 : 1;
}
#define TS_WIDTH_DISPATCH(T, B, CALL)           \
  do {                                          \
    switch (pack_width<T>(B)) {                 \
      case 4: { constexpr int W = 4; CALL; } break; \
      case 2: { constexpr int W = 2; CALL; } break; \
      default: { constexpr int W = 1; CALL; } break; \
    }                                           \
  } while (0)

// Partials of the last reduction -> (pointer, block count) for the finalize
// kernels. Distributed solves (ws.comm set) first sum the block partials and
// all-reduce the per-rank column sums, so every rank applies the reference's
// scalar logic to the same global numbers.
struct Partials {
  const double* p;
  int nblk;
};
Partials finish_partials(Workspace& ws, int nd, int32_t B, cudaStream_t s) {
  if (!ws.comm) return {ws.partial.get(), ws.nblk};
  k_sum_partials<<<1, kFinThreads, 0, s>>>(ws.partial.get(), nd, B, ws.nblk, ws.summed.get());
  TS_CUDA_LAUNCH();
  ws.comm->allreduce_sum(ws.summed.get(), size_t(nd) * B, s);
  return {ws.summed.get(), 1};
}

void check_batch(int32_t B) {
  if (B < 1 || B > kRedThreads) validation("batch must be in [1, 256]");
}

// Reduction grid for `len` entries: up to kRedBlocks (8 per SM) for the big levels, fewer for small
// vectors so the one-block finalize sums fewer partials. A function of len only: the block ranges,
// and so the summation order, are the same every call.
int red_grid(int64_t len) {
  const int64_t g = len / (int64_t(kRedThreads) * 32);
  return static_cast<int>(std::max<int64_t>(kRedMinBlocks, std::min<int64_t>(kRedBlocks, g)));
}

}  // namespace

void Workspace::ensure(int32_t batch) {
  partial.ensure(static_cast<size_t>(kRedBlocks) * 4 * batch);
  summed.ensure(static_cast<size_t>(4) * batch);
  if (!status.get()) {
    status.alloc(1);
    TS_CUDA(cudaMemset(status.get(), 0, sizeof(PcgStatus)));
    TS_CUDA(cudaMallocHost(&host_status, sizeof(PcgStatus)));
  }
}
Workspace::~Workspace() {
  if (host_status) cudaFreeHost(host_status);
}

template <typename T>
void dot2(const T* x0, const T* y0, const T* x1, const T* y1, int64_t ndof, int32_t batch, double* out,
          Workspace& ws, cudaStream_t s) {
  check_batch(batch);
  ws.ensure(batch);
  ws.nblk = red_grid(ndof * batch);
  TS_WIDTH_DISPATCH(T, batch, (k_dot2<T, W><<<ws.nblk, kRedThreads, 0, s>>>(x0, y0, x1, y1, ndof * batch, batch,
                                                                       ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  k_sum_partials<<<1, kFinThreads, 0, s>>>(ws.partial.get(), x1 ? 2 : 1, batch, ws.nblk, out);
  TS_CUDA_LAUNCH();
  if (ws.comm) ws.comm->allreduce_sum(out, size_t(x1 ? 2 : 1) * batch, s);
}
template void dot2<float>(const float*, const float*, const float*, const float*, int64_t, int32_t, double*,
                          Workspace&, cudaStream_t);
template void dot2<double>(const double*, const double*, const double*, const double*, int64_t, int32_t, double*,
                           Workspace&, cudaStream_t);

// beta from the (M^-1 e, e) partials the last init / update pass left behind
void pcg_rho(int32_t B, bool first, const ColScalars& cs, Workspace& ws, cudaStream_t s) {
  if (!ws.last_p) validation("pcg_rho: no (M^-1 e, e) partials pending");
  k_rho_final<<<1, kFinThreads, 0, s>>>(ws.last_p, ws.last_nd, ws.last_nd - 1, ws.last_nblk, B, first ? 1 : 0,
                                        cs[ColScalars::RHO_A], cs[ColScalars::RHO_B], cs[ColScalars::BETA]);
  TS_CUDA_LAUNCH();
  ws.last_p = nullptr;
}

template <typename T>
void pcg_direction(const T* inv, const T* e, T* p, int32_t n, int32_t B, bool first, const ColScalars& cs,
                   cudaStream_t s, T* q_init, const uint8_t* mask, T* u_pending) {
  if (u_pending && first) validation("pcg_direction: no previous direction to apply");
  TS_WIDTH_DISPATCH(T, B, (k_direction<T, W><<<grid_for(int64_t(n) * B / W, 256), 256, 0, s>>>(
                               inv, e, p, n, B, first ? 1 : 0, cs[ColScalars::BETA], q_init, mask, u_pending,
                               cs[ColScalars::ALPHA])));
  TS_CUDA_LAUNCH();
}

template <typename T>
void pcg_apply_pending(T* u, const T* p, int32_t n, int32_t B, const ColScalars& cs, cudaStream_t s) {
  TS_WIDTH_DISPATCH(T, B, (k_apply_pending<T, W><<<grid_for(3 * int64_t(n) * B / W, 256), 256, 0, s>>>(
                               u, p, n, B, cs[ColScalars::ALPHA])));
  TS_CUDA_LAUNCH();
}

template <typename T>
void pcg_gamma(const T* p, const T* q, int32_t n, int32_t B, const ColScalars& cs, Workspace& ws,
               cudaStream_t s) {
  ws.nblk = red_grid(3 * int64_t(n) * B);
  TS_WIDTH_DISPATCH(T, B, (k_gamma<T, W><<<ws.nblk, kRedThreads, 0, s>>>(p, q, 3 * int64_t(n) * B, B,
                                                                          ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 3, B, s);
  k_gamma_final<T><<<1, kFinThreads, 0, s>>>(pp.p, pp.nblk, B, cs[ColScalars::RHO_A], cs[ColScalars::RHO_B],
                                     cs[ColScalars::GAMMA], cs[ColScalars::ALPHA], ws.status.get());
  TS_CUDA_LAUNCH();
}

template <typename T>
void pcg_update(const T* inv, T* e, const T* q, int32_t n, int32_t B, const ColScalars& cs, Workspace& ws,
                cudaStream_t s) {
  ws.nblk = red_grid(int64_t(n) * B);
  TS_WIDTH_DISPATCH(T, B, (k_update<T, W><<<ws.nblk, kRedThreads, 0, s>>>(inv, e, q, n, B,
                                                                           cs[ColScalars::ALPHA], ws.status.get(),
                                                                           ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 2, B, s);
  k_ratio_final<<<1, kFinThreads, 0, s>>>(pp.p, 2, pp.nblk, B, cs[ColScalars::EN2], cs[ColScalars::RN2],
                                          ws.status.get());
  TS_CUDA_LAUNCH();
  ws.last_p = pp.p;
  ws.last_nblk = pp.nblk;
  ws.last_nd = 2;
}

template <typename T>
void pcg_init(const T* inv, const T* r, T* e, int32_t n, int32_t B, const ColScalars& cs, Workspace& ws,
              cudaStream_t s) {
  ws.nblk = red_grid(int64_t(n) * B);
  TS_WIDTH_DISPATCH(T, B, (k_init<T, W><<<ws.nblk, kRedThreads, 0, s>>>(inv, r, e, n, B, ws.partial.get(),
                                                                         ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 3, B, s);
  k_init_final<<<1, kFinThreads, 0, s>>>(pp.p, pp.nblk, B, cs[ColScalars::RN2], cs[ColScalars::EN2], ws.status.get());
  TS_CUDA_LAUNCH();
  ws.last_p = pp.p;
  ws.last_nblk = pp.nblk;
  ws.last_nd = 3;
}

#define INST(T)                                                                                              \
  template void pcg_direction<T>(const T*, const T*, T*, int32_t, int32_t, bool, const ColScalars&,         \
                                 cudaStream_t, T*, const uint8_t*, T*);                                      \
  template void pcg_apply_pending<T>(T*, const T*, int32_t, int32_t, const ColScalars&, cudaStream_t);       \
  template void pcg_gamma<T>(const T*, const T*, int32_t, int32_t, const ColScalars&, Workspace&,           \
                             cudaStream_t);                                                                  \
  template void pcg_update<T>(const T*, T*, const T*, int32_t, int32_t, const ColScalars&, Workspace&,       \
                              cudaStream_t);                                                                 \
  template void pcg_init<T>(const T*, const T*, T*, int32_t, int32_t, const ColScalars&, Workspace&,         \
                            cudaStream_t);                                                                   \
  template void bj_apply<T>(const T*, const T*, T*, int32_t, int32_t, cudaStream_t);
template <typename T>
void bj_apply(const T* inv, const T* r, T* z, int32_t n, int32_t B, cudaStream_t s) {
  k_bj_apply<T><<<grid_for(int64_t(n) * B, 256), 256, 0, s>>>(inv, r, z, n, B);
  TS_CUDA_LAUNCH();
}
INST(float)
INST(double)
#undef INST

void cg_true_residual(const double* f, double* r, int32_t n, int32_t B, const ColScalars& cs, Workspace& ws,
                      cudaStream_t s) {
  ws.nblk = red_grid(3 * int64_t(n) * B);
  TS_WIDTH_DISPATCH(double, B, (k_true_res<W><<<ws.nblk, kRedThreads, 0, s>>>(f, r, 3 * int64_t(n) * B, B,
                                                                               ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 1, B, s);
  k_ratio_final<<<1, kFinThreads, 0, s>>>(pp.p, 1, pp.nblk, B, cs[ColScalars::RN2], cs[ColScalars::FN2], ws.status.get());
  TS_CUDA_LAUNCH();
}

void cg_direction(const double* z, const double* q, double* p, int32_t n, int32_t B, bool first,
                  const ColScalars& cs, Workspace& ws, cudaStream_t s) {
  const int64_t len = 3 * int64_t(n) * B;
  if (!first) {
    ws.nblk = red_grid(len);
    TS_WIDTH_DISPATCH(double, B, (k_dot2<double, W><<<ws.nblk, kRedThreads, 0, s>>>(z, q, nullptr, nullptr, len, B,
                                                                                     ws.partial.get(), ws.owned)));
    TS_CUDA_LAUNCH();
    const Partials pp = finish_partials(ws, 1, B, s);
    k_cg_beta<<<1, kFinThreads, 0, s>>>(pp.p, pp.nblk, B, cs[ColScalars::GPREV], cs[ColScalars::BETA]);
    TS_CUDA_LAUNCH();
  }
  k_xpby<<<grid_for(len, 256), 256, 0, s>>>(z, p, len, B, first ? 1 : 0, cs[ColScalars::BETA]);
  TS_CUDA_LAUNCH();
}

void cg_alpha(const double* z, const double* r, const double* p, const double* q, int32_t n, int32_t B,
              const ColScalars& cs, Workspace& ws, cudaStream_t s) {
  ws.nblk = red_grid(3 * int64_t(n) * B);
  TS_WIDTH_DISPATCH(double, B, (k_dot2<double, W><<<ws.nblk, kRedThreads, 0, s>>>(z, r, p, q, 3 * int64_t(n) * B, B,
                                                                                   ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 2, B, s);
  k_cg_alpha<<<1, kFinThreads, 0, s>>>(pp.p, pp.nblk, B, cs[ColScalars::RHO_A], cs[ColScalars::GAMMA],
                               cs[ColScalars::GPREV], cs[ColScalars::ALPHA], ws.status.get());
  TS_CUDA_LAUNCH();
}

void cg_update(double* r, double* u, const double* p, const double* q, int32_t n, int32_t B, const ColScalars& cs,
               Workspace& ws, cudaStream_t s) {
  ws.nblk = red_grid(3 * int64_t(n) * B);
  TS_WIDTH_DISPATCH(double, B, (k_cg_update<W><<<ws.nblk, kRedThreads, 0, s>>>(r, u, p, q, 3 * int64_t(n) * B, B, cs[ColScalars::ALPHA],
                                                 ws.partial.get(), ws.owned)));
  TS_CUDA_LAUNCH();
  const Partials pp = finish_partials(ws, 1, B, s);
  k_ratio_final<<<1, kFinThreads, 0, s>>>(pp.p, 1, pp.nblk, B, cs[ColScalars::RN2], cs[ColScalars::FN2], ws.status.get());
  TS_CUDA_LAUNCH();
}

void bcsr_apply_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n, const float* u,
                    float* f, int32_t B, cudaStream_t s, int64_t nnz) {
  // fp64 row sums as the reference; W cases of a block row per thread, 16-byte u packs
  static const bool staged = [] {  // TSGPU_L2_STAGED=0: the unstaged kernel
    const char* e = std::getenv("TSGPU_L2_STAGED");
    return !e || std::atoi(e) != 0;
  }();
  if (n > 0 && staged && nnz > 0 && pack_width<float>(B) == 4 && (B == 16 || B == 8)) {
    // capacity 24 blocks per row; r = 8 as two cases per thread over four threads per row
    // (measured at configs[2] size: level-2 solve time r = 8 0.218 -> 0.175 s, r = 16 unchanged)
    if (B == 16) launch_rows_staged<4, 8, double, 24>(row_ptr, col_idx, blocks, n, nnz, u, f, B, s);
    else launch_rows_staged<2, 8, double, 24>(row_ptr, col_idx, blocks, n, nnz, u, f, B, s);
    TS_CUDA_LAUNCH();
    return;
  }
  TS_WIDTH_DISPATCH(float, B, (k_bcsr_rows<W, double><<<grid_for(int64_t(n) * (B / W), 256), 256, 0, s>>>(
                                   row_ptr, col_idx, blocks, n, u, f, B, nullptr)));
  TS_CUDA_LAUNCH();
}
bool bcsr_rows_staged_ok(int32_t B) {
  static const bool staged = [] {  // TSGPU_L1_STAGED=0: the unstaged kernel for every product
    const char* e = std::getenv("TSGPU_L1_STAGED");
    return !e || std::atoi(e) != 0;
  }();
  return staged && pack_width<float>(B) == 4 && (B == 16 || B == 8);
}
void bcsr_rows_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n, const float* u,
                   float* f, int32_t B, cudaStream_t s, const int32_t* rows, int64_t nnz) {
  if (n <= 0) return;
  if (!rows && nnz > 0 && bcsr_rows_staged_ok(B)) {
    // capacity 16 blocks per row (+8 per warp): a box mesh's rows have at most 15; the smaller
    // staging leaves more of the unified L1 to the u gathers (measured: PER_ROW 20 -> 16 is
    // 0.568 -> 0.484 ms at r = 16). r = 8: two cases per thread and four threads per row (8 rows
    // per warp) beat four cases per thread (16 rows per warp: twice the staging per warp).
    if (B == 16) launch_rows_staged<4, 8, float, 16>(row_ptr, col_idx, blocks, n, nnz, u, f, B, s);
    else launch_rows_staged<2, 8, float, 16>(row_ptr, col_idx, blocks, n, nnz, u, f, B, s);
    TS_CUDA_LAUNCH();
    return;
  }
  TS_WIDTH_DISPATCH(float, B, (k_bcsr_rows<W, float><<<grid_for(int64_t(n) * (B / W), 256), 256, 0, s>>>(
                                   row_ptr, col_idx, blocks, n, u, f, B, rows)));
  TS_CUDA_LAUNCH();
}
bool bcsr_rows_f32_gamma(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n,
                         const float* p, float* q, int32_t B, cudaStream_t s, int64_t nnz, Workspace& ws,
                         const uint8_t* rowsel) {
  static const bool on = [] {  // TSGPU_L1_FUSED_DOTS=0: the product, then the separate gamma pass
    const char* e = std::getenv("TSGPU_L1_FUSED_DOTS");
    return !e || e[0] != '0';
  }();
  if (!on || n <= 0 || nnz <= 0 || !bcsr_rows_staged_ok(B)) return false;
  if (!rowsel && (ws.comm || ws.owned)) return false;  // partitioned callers select their rows
  ws.ensure(B);
  const int grid = B == 16 ? launch_rows_staged<4, 8, float, 16, true>(row_ptr, col_idx, blocks, n, nnz, p, q, B, s,
                                                                        ws.partial.get(), rowsel)
                           : launch_rows_staged<2, 8, float, 16, true>(row_ptr, col_idx, blocks, n, nnz, p, q, B, s,
                                                                        ws.partial.get(), rowsel);
  TS_CUDA_LAUNCH();
  ws.nblk = grid;
  return true;
}

bool bcsr_apply_f32_gamma(const int32_t* row_ptr, const int32_t* col_idx, const float* blocks, int32_t n,
                          const float* p, float* q, int32_t B, cudaStream_t s, int64_t nnz, Workspace& ws) {
  static const bool on = [] {  // TSGPU_L2_FUSED_DOTS=0: the product, then the separate gamma pass
    const char* e = std::getenv("TSGPU_L2_FUSED_DOTS");
    return !e || e[0] != '0';
  }();
  static const bool staged = [] {
    const char* e = std::getenv("TSGPU_L2_STAGED");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || !staged || n <= 0 || nnz <= 0 || ws.comm || ws.owned || pack_width<float>(B) != 4 ||
      (B != 16 && B != 8))
    return false;
  ws.ensure(B);
  const int grid = B == 16 ? launch_rows_staged<4, 8, double, 24, true>(row_ptr, col_idx, blocks, n, nnz, p, q, B, s,
                                                                         ws.partial.get())
                           : launch_rows_staged<2, 8, double, 24, true>(row_ptr, col_idx, blocks, n, nnz, p, q, B, s,
                                                                         ws.partial.get());
  TS_CUDA_LAUNCH();
  ws.nblk = grid;
  return true;
}

// (p,q), (p,p), (q,q) per column over the listed node rows, into partial rows [ws.nblk, ...): the
// rows the fused product left out (a partition's interface rows, complete only after the exchange)
__global__ void __launch_bounds__(256) k_rows_dots(const float* __restrict__ p, const float* __restrict__ q,
                                                   const int32_t* __restrict__ rows, int32_t n, int32_t B,
                                                   double* __restrict__ partial) {
  __shared__ double sm[3][256];
  const int t = threadIdx.x, per = 256 / B, col = t % B, slot = t / B;
  double a = 0.0, b = 0.0, c = 0.0;
  if (slot < per)
    for (int64_t i = int64_t(blockIdx.x) * per + slot; i < n; i += int64_t(gridDim.x) * per) {
      const int64_t base = 3 * int64_t(__ldg(rows + i)) * B + col;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double x = double(p[base + d * B]), y = double(q[base + d * B]);
        a += x * y;
        b += x * x;
        c += y * y;
      }
    }
  sm[0][t] = slot < per ? a : 0.0;
  sm[1][t] = slot < per ? b : 0.0;
  sm[2][t] = slot < per ? c : 0.0;
  __syncthreads();
  if (t < B)
    for (int k = 0; k < 3; ++k) {
      double sum = 0.0;
      for (int j = 0; j < per; ++j) sum += sm[k][j * B + t];
      partial[(int64_t(blockIdx.x) * 3 + k) * B + t] = sum;
    }
}

void rows_dots_append(const float* p, const float* q, const int32_t* rows, int32_t n, int32_t B, cudaStream_t s,
                      Workspace& ws) {
  if (n <= 0) return;
  const int per = 256 / B;
  const int nb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kRedBlocks - ws.nblk,
                                                                        (int64_t(n) + 8 * per - 1) / (8 * per))));
  k_rows_dots<<<nb, 256, 0, s>>>(p, q, rows, n, B, ws.partial.get() + int64_t(ws.nblk) * 3 * B);
  TS_CUDA_LAUNCH();
  ws.nblk += nb;
}

template <typename T>
void pcg_gamma_final(int32_t B, const ColScalars& cs, Workspace& ws, cudaStream_t s, bool partial_pq_only) {
  const Partials pp = finish_partials(ws, 3, B, s);
  static const bool force_fallback = [] {
    const char* e = std::getenv("TSGPU_TEST_FUSED_FALLBACK");
    return e && e[0] == '1';
  }();
  k_gamma_final<T><<<1, kFinThreads, 0, s>>>(pp.p, pp.nblk, B, cs[ColScalars::RHO_A], cs[ColScalars::RHO_B],
                                     cs[ColScalars::GAMMA], cs[ColScalars::ALPHA], ws.status.get(),
                                     partial_pq_only ? (force_fallback ? 2 : 1) : 0);
  TS_CUDA_LAUNCH();
}
template void pcg_gamma_final<float>(int32_t, const ColScalars&, Workspace&, cudaStream_t, bool);
template void pcg_gamma_final<double>(int32_t, const ColScalars&, Workspace&, cudaStream_t, bool);

void cast_d2f(const double* x, float* y, int64_t n, cudaStream_t s) {
  k_cast_d2f<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
  TS_CUDA_LAUNCH();
}
void cast_f2d(const float* x, double* y, int64_t n, cudaStream_t s) {
  k_cast_f2d<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
  TS_CUDA_LAUNCH();
}
void zero_masked_f32(float* x, const uint8_t* mask, int64_t ndof, int32_t B, cudaStream_t s) {
  if (!mask) return;
  k_zero_masked<<<grid_for(ndof * B, 256), 256, 0, s>>>(x, mask, ndof * B, B);
  TS_CUDA_LAUNCH();
}
void p1_apply(const float* coarse, float* fine, const int32_t* edge_ends, int32_t nv, int32_t nf,
              const uint8_t* fine_mask, int32_t B, cudaStream_t s) {
  k_p1_apply<<<grid_for(3 * int64_t(nf) * B, 256), 256, 0, s>>>(coarse, fine, edge_ends, nv, nf, fine_mask, B);
  TS_CUDA_LAUNCH();
}
void p1_restrict(const float* fine, float* coarse, const int32_t* t_ptr, const int32_t* t_idx, int32_t nv,
                 const uint8_t* coarse_mask, int32_t B, cudaStream_t s, const uint8_t* owned) {
  k_p1_restrict<<<grid_for(3 * int64_t(nv) * B, 256), 256, 0, s>>>(fine, coarse, t_ptr, t_idx, nv, coarse_mask, B,
                                                                  owned);
  TS_CUDA_LAUNCH();
}
void p2_apply(const float* coarse, float* fine, const int32_t* agg, int32_t nf, const uint8_t* fine_mask, int32_t B,
              cudaStream_t s) {
  k_p2_apply<<<grid_for(3 * int64_t(nf) * B, 256), 256, 0, s>>>(coarse, fine, agg, nf, fine_mask, B);
  TS_CUDA_LAUNCH();
}
void p2_restrict(const float* fine, float* coarse, const int32_t* a_ptr, const int32_t* a_idx, int32_t nc,
                 const uint8_t* coarse_mask, int32_t B, cudaStream_t s) {
  k_p2_restrict<<<grid_for(3 * int64_t(nc) * B, 256), 256, 0, s>>>(fine, coarse, a_ptr, a_idx, nc, coarse_mask, B);
  TS_CUDA_LAUNCH();
}

}  // namespace tsg
