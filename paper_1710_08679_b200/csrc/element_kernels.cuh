// element_kernels.cuh — flop-lean exact element products for straight-sided
// tet10 / tet4 linear elasticity, evaluated per lane vector of load cases.
//
// Reference semantics: f_e = K_e u_e with K_e the 30x30 (tet10) or 12x12
// (tet4) stiffness of detail::tet10_stiffness_kernel / tet4_stiffness_kernel
// (element_stiffness.hpp:104-140). The reference rebuilds K_e (~26k flops)
// and multiplies it densely (1800 flops per case). Here the same exact
// integral is evaluated without forming K_e:
//
//   b_k = grad L_k (k = 1..3, b_0 = -(b_1+b_2+b_3)), constant per element.
//   tet10: grad u is linear, so it is fixed by its values G_i at the 4
//   vertices:  G_i = sum_{k=1..3} E_ik b_k^T with integer-coefficient nodal
//   combinations E_ik (below). sigma is linear too: S_i = lambda tr(G_i) I
//   + mu (G_i + G_i^T). With int L_i L_j dV = V (1 + delta_ij) / 20 the
//   weak form becomes  f = E^T [ (S_j + sum_i S_i) (V/20) b_k ]  — the exact
//   integral the reference's 4-point rule (exact for this quadratic
//   integrand, element_stiffness.hpp:35-51) also computes.
//   tet4: constant strain, f_a = V sigma b_a.
//
// Cost per load case: ~480 flops (tet10) / ~85 flops (tet4), all FFMA2 /
// FADD2 / FMUL2 for fp32 pairs. Validated against the reference K_e to
// 1.8e-15 relative (tests/test_element_formulation.py).
//
// Per-element coefficient record (12 scalars of T): b_1, b_2, b_3 (row k =
// d/dx,y,z of L_k), lp, mp, pad with lp = lambda V / 20, mp = mu V / 20 for
// tet10 and lp = lambda V, mp = mu V for tet4.
#pragma once
#include "lane_ops.cuh"

namespace tsg {

// S' from G (row c = component, col d = derivative): 6 values xx yy zz xy yz zx
template <class V>
__device__ __forceinline__ void stress6(const V (&G)[3][3], V lp, V mp2, V mp, V (&s)[6]) {
  using O = LaneOps<V>;
  const V tr = O::add(O::add(G[0][0], G[1][1]), G[2][2]);
  const V ltr = O::mul(lp, tr);
  s[0] = O::fma(mp2, G[0][0], ltr);
  s[1] = O::fma(mp2, G[1][1], ltr);
  s[2] = O::fma(mp2, G[2][2], ltr);
  s[3] = O::mul(mp, O::add(G[0][1], G[1][0]));
  s[4] = O::mul(mp, O::add(G[1][2], G[2][1]));
  s[5] = O::mul(mp, O::add(G[2][0], G[0][2]));
}

// G[c][d] = sum_k E[c][k] * b[k][d]
template <class V>
__device__ __forceinline__ void grad_from(const V (&E)[3][3], const V (&b)[3][3], V (&G)[3][3]) {
  using O = LaneOps<V>;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      G[c][d] = O::fma(E[c][2], b[2][d], O::fma(E[c][1], b[1][d], O::mul(E[c][0], b[0][d])));
}

// H = S b (symmetric S in 6-value form)
template <class V>
__device__ __forceinline__ void sym_mul(const V (&s)[6], const V (&bk)[3], V (&h)[3]) {
  using O = LaneOps<V>;
  h[0] = O::fma(s[5], bk[2], O::fma(s[3], bk[1], O::mul(s[0], bk[0])));
  h[1] = O::fma(s[4], bk[2], O::fma(s[1], bk[1], O::mul(s[3], bk[0])));
  h[2] = O::fma(s[2], bk[2], O::fma(s[4], bk[1], O::mul(s[5], bk[0])));
}

// tet10: u[a][c] (local node a in reference order, component c) -> f[a][c]
template <class V>
__device__ __forceinline__ void tet10_product(const V (&u)[10][3], const V (&b)[3][3], V lp, V mp,
                                              V (&f)[10][3]) {
  using O = LaneOps<V>;
  const V three = O::splat(3), four = O::splat(4), mfour = O::splat(-4), mthree = O::splat(-3);
  const V mp2 = O::add(mp, mp);
  // edge nodes: 4=(0,1) 5=(1,2) 6=(2,0) 7=(0,3) 8=(1,3) 9=(2,3)
  V S[4][6];
  {
    V E[3][3];  // vertex 0: E_0k = 4 u_0k + (-3 u_0 - u_k)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V m = O::mul(mthree, u[0][c]);
      E[c][0] = O::fma(four, u[4][c], O::sub(m, u[1][c]));
      E[c][1] = O::fma(four, u[6][c], O::sub(m, u[2][c]));
      E[c][2] = O::fma(four, u[7][c], O::sub(m, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[0]);
  }
  {
    V E[3][3];  // vertex 1: s = u_0 - 4 u_01 ; E_11 = 3u_1 + s ; E_12 = 4u_12 - u_2 + s ; E_13 = 4u_13 - u_3 + s
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[4][c], u[0][c]);
      E[c][0] = O::fma(three, u[1][c], s);
      E[c][1] = O::fma(four, u[5][c], O::sub(s, u[2][c]));
      E[c][2] = O::fma(four, u[8][c], O::sub(s, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[1]);
  }
  {
    V E[3][3];  // vertex 2: s = u_0 - 4 u_02 ; E_21 = 4u_21 - u_1 + s ; E_22 = 3u_2 + s ; E_23 = 4u_23 - u_3 + s
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[6][c], u[0][c]);
      E[c][0] = O::fma(four, u[5][c], O::sub(s, u[1][c]));
      E[c][1] = O::fma(three, u[2][c], s);
      E[c][2] = O::fma(four, u[9][c], O::sub(s, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[2]);
  }
  {
    V E[3][3];  // vertex 3: s = u_0 - 4 u_03 ; E_31 = 4u_31 - u_1 + s ; E_32 = 4u_32 - u_2 + s ; E_33 = 3u_3 + s
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[7][c], u[0][c]);
      E[c][0] = O::fma(four, u[8][c], O::sub(s, u[1][c]));
      E[c][1] = O::fma(four, u[9][c], O::sub(s, u[2][c]));
      E[c][2] = O::fma(three, u[3][c], s);
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[3]);
  }
  V Ssum[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) Ssum[q] = O::add(O::add(S[0][q], S[1][q]), O::add(S[2][q], S[3][q]));

  // f = E^T H, H_jk = (S_j + sum_i S_i)(V/20) b_k, T_j = sum_k H_jk, accumulated per j:
  //   f0 = -3 T0 + T1 + T2 + T3          f1 = -H01 + 3 H11 - H21 - H31
  //   f2 = -H02 - H12 + 3 H22 - H32      f3 = -H03 - H13 - H23 + 3 H33
  //   f4 = 4 (H01 - T1)  f6 = 4 (H02 - T2)  f7 = 4 (H03 - T3)
  //   f5 = 4 (H12 + H21)  f8 = 4 (H13 + H31)  f9 = 4 (H23 + H32)
  // The negated sums ride in FFMA2 operand signs (O::neg), so no separate negations.
  V t0[3], s0[3];
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[0][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      t0[c] = O::add(O::add(h1[c], h2[c]), h3[c]);
      f[4][c] = O::mul(four, h1[c]);
      f[6][c] = O::mul(four, h2[c]);
      f[7][c] = O::mul(four, h3[c]);
      f[1][c] = h1[c];  // +H01 (negated below)
      f[2][c] = h2[c];  // +H02 ...
      f[3][c] = h3[c];  // +H03 ...
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[1][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      s0[c] = t;
      f[4][c] = O::fma(mfour, t, f[4][c]);
      f[1][c] = O::fma(three, h1[c], O::neg(f[1][c]));  // 3 H11 - H01
      f[5][c] = O::mul(four, h2[c]);
      f[2][c] = O::add(f[2][c], h2[c]);                 // H02 + H12
      f[8][c] = O::mul(four, h3[c]);
      f[3][c] = O::add(f[3][c], h3[c]);                 // H03 + H13
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[2][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      s0[c] = O::add(s0[c], t);
      f[6][c] = O::fma(mfour, t, f[6][c]);
      f[5][c] = O::fma(four, h1[c], f[5][c]);
      f[1][c] = O::sub(f[1][c], h1[c]);
      f[2][c] = O::fma(three, h2[c], O::neg(f[2][c]));  // 3 H22 - H02 - H12
      f[9][c] = O::mul(four, h3[c]);
      f[3][c] = O::add(f[3][c], h3[c]);                 // H03 + H13 + H23
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[3][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      f[0][c] = O::fma(mthree, t0[c], O::add(s0[c], t));
      f[7][c] = O::fma(mfour, t, f[7][c]);
      f[8][c] = O::fma(four, h1[c], f[8][c]);
      f[1][c] = O::sub(f[1][c], h1[c]);
      f[9][c] = O::fma(four, h2[c], f[9][c]);
      f[2][c] = O::sub(f[2][c], h2[c]);
      f[3][c] = O::fma(three, h3[c], O::neg(f[3][c]));  // 3 H33 - H03 - H13 - H23
    }
  }
}

// tet10 product writing through an accessor F(s, c) -> V& (compile-time slot s,
// component c) that ACCUMULATES into the slots of the bit mask ACC (the rest are
// overwritten). Same operations as tet10_product; an accumulated slot costs at
// most one extra op per component (the first write of slots 0-3 becomes a
// subtraction / addition; slots 4-9 fold into the FMA that first writes them).
// Used by the fan sweep (ebe_fan.cu), where rows shared with the previous element
// of the fan keep their partial sums in registers.
template <unsigned ACC, class V, class F>
__device__ __forceinline__ void tet10_product_acc(const V (&u)[10][3], const V (&b)[3][3], V lp, V mp, F&& fr) {
  using O = LaneOps<V>;
  constexpr bool A0 = ACC & 1u, A1 = ACC & 2u, A2 = ACC & 4u, A3 = ACC & 8u, A4 = ACC & 16u, A5 = ACC & 32u,
                 A6 = ACC & 64u, A7 = ACC & 128u, A8 = ACC & 256u, A9 = ACC & 512u;
  const V three = O::splat(3), four = O::splat(4), mfour = O::splat(-4), mthree = O::splat(-3);
  const V mp2 = O::add(mp, mp);
  V S[4][6];
  {
    V E[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V m = O::mul(mthree, u[0][c]);
      E[c][0] = O::fma(four, u[4][c], O::sub(m, u[1][c]));
      E[c][1] = O::fma(four, u[6][c], O::sub(m, u[2][c]));
      E[c][2] = O::fma(four, u[7][c], O::sub(m, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[0]);
  }
  {
    V E[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[4][c], u[0][c]);
      E[c][0] = O::fma(three, u[1][c], s);
      E[c][1] = O::fma(four, u[5][c], O::sub(s, u[2][c]));
      E[c][2] = O::fma(four, u[8][c], O::sub(s, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[1]);
  }
  {
    V E[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[6][c], u[0][c]);
      E[c][0] = O::fma(four, u[5][c], O::sub(s, u[1][c]));
      E[c][1] = O::fma(three, u[2][c], s);
      E[c][2] = O::fma(four, u[9][c], O::sub(s, u[3][c]));
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[2]);
  }
  {
    V E[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V s = O::fma(mfour, u[7][c], u[0][c]);
      E[c][0] = O::fma(four, u[8][c], O::sub(s, u[1][c]));
      E[c][1] = O::fma(four, u[9][c], O::sub(s, u[2][c]));
      E[c][2] = O::fma(three, u[3][c], s);
    }
    V G[3][3];
    grad_from(E, b, G);
    stress6(G, lp, mp2, mp, S[3]);
  }
  V Ssum[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) Ssum[q] = O::add(O::add(S[0][q], S[1][q]), O::add(S[2][q], S[3][q]));
  // first writes: accumulated slots 1-3 hold (H - acc), so the negations below give (acc - H)
  V t0[3], s0[3];
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[0][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      t0[c] = O::add(O::add(h1[c], h2[c]), h3[c]);
      fr(4, c) = A4 ? O::fma(four, h1[c], fr(4, c)) : O::mul(four, h1[c]);
      fr(6, c) = A6 ? O::fma(four, h2[c], fr(6, c)) : O::mul(four, h2[c]);
      fr(7, c) = A7 ? O::fma(four, h3[c], fr(7, c)) : O::mul(four, h3[c]);
      fr(1, c) = A1 ? O::sub(h1[c], fr(1, c)) : h1[c];
      fr(2, c) = A2 ? O::sub(h2[c], fr(2, c)) : h2[c];
      fr(3, c) = A3 ? O::sub(h3[c], fr(3, c)) : h3[c];
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[1][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      s0[c] = t;
      fr(4, c) = O::fma(mfour, t, fr(4, c));
      fr(1, c) = O::fma(three, h1[c], O::neg(fr(1, c)));
      fr(5, c) = A5 ? O::fma(four, h2[c], fr(5, c)) : O::mul(four, h2[c]);
      fr(2, c) = O::add(fr(2, c), h2[c]);
      fr(8, c) = A8 ? O::fma(four, h3[c], fr(8, c)) : O::mul(four, h3[c]);
      fr(3, c) = O::add(fr(3, c), h3[c]);
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[2][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      s0[c] = O::add(s0[c], t);
      fr(6, c) = O::fma(mfour, t, fr(6, c));
      fr(5, c) = O::fma(four, h1[c], fr(5, c));
      fr(1, c) = O::sub(fr(1, c), h1[c]);
      fr(2, c) = O::fma(three, h2[c], O::neg(fr(2, c)));
      fr(9, c) = A9 ? O::fma(four, h3[c], fr(9, c)) : O::mul(four, h3[c]);
      fr(3, c) = O::add(fr(3, c), h3[c]);
    }
  }
  {
    V sh[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[q] = O::add(S[3][q], Ssum[q]);
    V h1[3], h2[3], h3[3];
    sym_mul(sh, b[0], h1);
    sym_mul(sh, b[1], h2);
    sym_mul(sh, b[2], h3);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V t = O::add(O::add(h1[c], h2[c]), h3[c]);
      fr(0, c) = A0 ? O::fma(mthree, t0[c], O::add(O::add(s0[c], t), fr(0, c)))
                    : O::fma(mthree, t0[c], O::add(s0[c], t));
      fr(7, c) = O::fma(mfour, t, fr(7, c));
      fr(8, c) = O::fma(four, h1[c], fr(8, c));
      fr(1, c) = O::sub(fr(1, c), h1[c]);
      fr(9, c) = O::fma(four, h2[c], fr(9, c));
      fr(2, c) = O::sub(fr(2, c), h2[c]);
      fr(3, c) = O::fma(three, h3[c], O::neg(fr(3, c)));
    }
  }
}

// tet4 (constant strain): G = sum_k (u_k - u_0) b_k^T ; f_k = V sigma b_k ; f_0 = -sum f_k
template <class V>
__device__ __forceinline__ void tet4_product(const V (&u)[4][3], const V (&b)[3][3], V lp, V mp,
                                             V (&f)[4][3]) {
  using O = LaneOps<V>;
  V E[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < 3; ++k) E[c][k] = O::sub(u[k + 1][c], u[0][c]);
  V G[3][3];
  grad_from(E, b, G);
  V s[6];
  stress6(G, lp, O::add(mp, mp), mp, s);
  V h[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) sym_mul(s, b[k], h[k]);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    f[1][c] = h[0][c];
    f[2][c] = h[1][c];
    f[3][c] = h[2][c];
    f[0][c] = O::sub(O::zero(), O::add(O::add(h[0][c], h[1][c]), h[2][c]));
  }
}

}  // namespace tsg
