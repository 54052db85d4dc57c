"""The device kernels evaluate K_e u_e without forming K_e (element_kernels.cuh).

This CPU test re-derives that flop-lean formulation in numpy and checks it
against the oracle's element matrices (detail::tet10_stiffness_kernel /
tet4_stiffness_kernel, element_stiffness.hpp:104-140) on random shapes:
the vertex-moment form is the exact integral, so agreement is to rounding.
"""
import numpy as np


def lean_tet10(v, lam, mu, u):
    J = np.stack([v[k + 1] - v[0] for k in range(3)], axis=1)
    inv = np.linalg.inv(J)
    V = np.linalg.det(J) / 6
    b = [None, inv[0], inv[1], inv[2]]
    lp, mp = lam * V / 20, mu * V / 20
    u0, u1, u2, u3, u4, u5, u6, u7, u8, u9 = u
    t0 = 3 * u0
    s1, s2, s3 = u0 - 4 * u4, u0 - 4 * u6, u0 - 4 * u7
    E = {(0, 1): 4 * u4 - u1 - t0, (0, 2): 4 * u6 - u2 - t0, (0, 3): 4 * u7 - u3 - t0,
         (1, 1): 3 * u1 + s1, (1, 2): 4 * u5 - u2 + s1, (1, 3): 4 * u8 - u3 + s1,
         (2, 1): 4 * u5 - u1 + s2, (2, 2): 3 * u2 + s2, (2, 3): 4 * u9 - u3 + s2,
         (3, 1): 4 * u8 - u1 + s3, (3, 2): 4 * u9 - u2 + s3, (3, 3): 3 * u3 + s3}
    S = []
    for i in range(4):
        G = sum(np.outer(E[(i, k)], b[k]) for k in (1, 2, 3))
        S.append(lp * np.trace(G) * np.eye(3) + mp * (G + G.T))
    Ssum = sum(S)
    H = {(j, k): (S[j] + Ssum) @ b[k] for j in range(4) for k in (1, 2, 3)}
    T = [sum(H[(i, k)] for k in (1, 2, 3)) for i in range(4)]
    f = np.zeros((10, 3))
    f[0] = -3 * T[0] + T[1] + T[2] + T[3]
    f[4], f[6], f[7] = 4 * (H[(0, 1)] - T[1]), 4 * (H[(0, 2)] - T[2]), 4 * (H[(0, 3)] - T[3])
    f[5], f[8], f[9] = 4 * (H[(1, 2)] + H[(2, 1)]), 4 * (H[(1, 3)] + H[(3, 1)]), 4 * (H[(2, 3)] + H[(3, 2)])
    f[1] = 3 * H[(1, 1)] - H[(0, 1)] - H[(2, 1)] - H[(3, 1)]
    f[2] = 3 * H[(2, 2)] - H[(0, 2)] - H[(1, 2)] - H[(3, 2)]
    f[3] = 3 * H[(3, 3)] - H[(0, 3)] - H[(1, 3)] - H[(2, 3)]
    return f


def lean_tet4(v, lam, mu, u):
    J = np.stack([v[k + 1] - v[0] for k in range(3)], axis=1)
    inv = np.linalg.inv(J)
    V = np.linalg.det(J) / 6
    b = [-(inv[0] + inv[1] + inv[2]), inv[0], inv[1], inv[2]]
    G = sum(np.outer(u[k] - u[0], b[k]) for k in (1, 2, 3))
    S = lam * V * np.trace(G) * np.eye(3) + mu * V * (G + G.T)
    return np.array([S @ b[k] for k in range(4)])


def test_lean_products_match_reference_element_matrices(port):
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(40):
        v = rng.standard_normal((4, 3))
        if np.linalg.det(np.stack([v[k + 1] - v[0] for k in range(3)], 1)) < 0:
            v[[2, 3]] = v[[3, 2]]
        lam, mu = rng.uniform(1, 3), rng.uniform(1, 3)
        K10 = port.element_matrix(2, v.ravel(), lam, mu)
        u = rng.standard_normal((10, 3))
        ref = (K10 @ u.ravel()).reshape(10, 3)
        worst = max(worst, np.abs(lean_tet10(v, lam, mu, u) - ref).max() / np.abs(ref).max())
        K4 = port.element_matrix(1, v.ravel(), lam, mu)
        u4 = rng.standard_normal((4, 3))
        ref4 = (K4 @ u4.ravel()).reshape(4, 3)
        worst = max(worst, np.abs(lean_tet4(v, lam, mu, u4) - ref4).max() / np.abs(ref4).max())
    assert worst < 1e-13
