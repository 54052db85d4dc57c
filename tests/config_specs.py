"""BASELINE.json configs as test inputs (shared by the GPU parity tests and the
fixture generators under tests/golden/).

configs[0]: the small cube the CPU reference solves in full (SURVEY §6.2 probe:
            8^3 cells, extents 8, one interface at 4, Table-3 two-layer set).
configs[1]: the 10M-DOF layered-crust box of the matvec microbenchmark
            (82 x 123 x 41 cells of 2.8 km; bench.py mesh_spec).
configs[2]: the 50M-DOF 3-layer crust box (140 x 210 x 70 cells; bench.py
            solve leg).
"""
import numpy as np

CELL_KM = 2.8
TWO_LAYER = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0)]  # Table 3
THREE_LAYER = TWO_LAYER + [(6800.0, 3900.0, 2900.0)]  # 3rd layer invented (vp^2 > 2 vs^2)


def lame(table):
    lam = np.array([rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in table])
    mu = np.array([rho * vs * vs for vp, vs, rho in table])
    return lam, mu


CONFIG0 = dict(extents=(8.0, 8.0, 8.0), cells=(8, 8, 8), interfaces=(4.0,), table=TWO_LAYER, batch=4)
CONFIG1 = dict(cells=(82, 123, 41), extents=lambda c: tuple(x * CELL_KM * 1e3 for x in c),
               interfaces=lambda c: (0.75 * c[2] * CELL_KM * 1e3,), table=TWO_LAYER)
CONFIG2 = dict(cells=(140, 210, 70), extents=lambda c: tuple(x * CELL_KM * 1e3 for x in c),
               interfaces=lambda c: (0.4 * c[2] * CELL_KM * 1e3, 0.75 * c[2] * CELL_KM * 1e3),
               table=THREE_LAYER, batch=4)


def smooth_batch(orc, coords, extents, mask, batch, seed=31):
    """acceptance_main.cpp:82-102 smooth fields: one field per column with
    amplitude 0.05 (1 + 0.2 sym) and ky in {1, 2} from DeterministicRng(seed)."""
    r = orc.rng_sym(seed, 2 * batch)
    x, y, z = (coords[:, k] / extents[k] for k in range(3))
    sz = np.sin(0.5 * np.pi * z)
    u = np.empty((coords.shape[0], 3, batch))
    for b in range(batch):
        amp = 0.05 * (1.0 + 0.2 * r[2 * b])
        ky = 1.0 + (0.0 if (r[2 * b + 1] + 1) / 2 < 0.5 else 1.0)
        cx, sx = np.cos(np.pi * x), np.sin(np.pi * x)
        cy, sy = np.cos(ky * np.pi * y), np.sin(ky * np.pi * y)
        u[:, 0, b] = amp * sx * cy * sz
        u[:, 1, b] = amp * cx * sy * sz
        u[:, 2, b] = amp * cx * cy * sz
    u = u.reshape(-1, batch)
    u[np.asarray(mask) == 1] = 0.0
    return u


def config2_rhs(orc, coords, extents, mask, batch):
    return smooth_batch(orc, coords, extents, mask, batch, seed=31)
