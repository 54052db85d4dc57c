"""Pin the C restatement oracle (oracle/tsoracle.c) before trusting it.

1. Against the UNMODIFIED reference compiled in place (oracle/_ref/libtsref.so):
   bit-exact on meshes, element matrices, EBE products (both tiers, both
   orders), assembly, block Jacobi, transfers, aggregation + level-2 Galerkin
   product, inner PCG, full multigrid solve() and solve_pcge().
2. Against the committed golden fixtures (tests/golden/, generated from the
   reference by tests/golden/make_golden.py) — this leg runs everywhere,
   including the GPU box where /root/reference is absent.
"""
import os

import numpy as np
import pytest
from conftest import STIFF, TWO_LAYER, lame

from oracle import MeshArrays, SolverConfig

GOLD = os.path.join(os.path.dirname(__file__), "golden")

MESHES = [
    ((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1),
    ((400.0, 400.0, 200.0), (3, 3, 2), (100.0,), 1),
    ((1.0, 2.0, 3.0), (3, 2, 1), (1.0, 2.0), 2),
    ((1.0, 1.0, 1.0), (1, 1, 1), (), 0),
]


@pytest.mark.parametrize("spec", MESHES)
def test_box_mesh_bit_exact(port, reference, spec):
    a, b = port.box_mesh(*spec), reference.box_mesh(*spec)
    assert a.vertex_count == b.vertex_count
    for k in ("coords", "tets10", "material_id", "bc_node", "bc_axis"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_rng_stream(port, reference):
    assert np.array_equal(port.rng_sym(2024, 5000), reference.rng_sym(2024, 5000))


@pytest.mark.parametrize("order", [1, 2])
def test_element_matrix_bit_exact(port, reference, order):
    rng = np.random.default_rng(3)
    for _ in range(5):
        v = rng.standard_normal((4, 3))
        ka = port.element_matrix(order, v.ravel(), 2.5, 1.5)
        kb = reference.element_matrix(order, v.ravel(), 2.5, 1.5)
        assert np.array_equal(ka, kb)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("masked", [True, False])
def test_operators_bit_exact(port, reference, prec, order, masked):
    m = reference.box_mesh((400.0, 400.0, 200.0), (3, 3, 2), (100.0,), 1)
    lam, mu = lame(TWO_LAYER)
    nn = m.vertex_count if order == 1 else m.n_nodes
    mask = m.dirichlet_mask()[: 3 * nn] if masked else None
    u = reference.rng_sym(11, 3 * nn * 5).reshape(3 * nn, 5)
    assert np.array_equal(port.ebe_apply(m, order, lam, mu, mask, prec, u),
                          reference.ebe_apply(m, order, lam, mu, mask, prec, u))
    A = port.assemble_bcsr(m, order, lam, mu, mask, prec)
    B = reference.assemble_bcsr(m, order, lam, mu, mask, prec)
    for x, y in zip(A, B):
        assert np.array_equal(x, y)
    assert np.array_equal(port.bcsr_apply(A[0], A[1], A[2], prec, u), reference.bcsr_apply(B[0], B[1], B[2], prec, u))
    if masked or order == 2:
        ia = port.ebe_block_jacobi(m, order, lam, mu, mask if masked else m.dirichlet_mask()[: 3 * nn], prec)
        ib = reference.ebe_block_jacobi(m, order, lam, mu, mask if masked else m.dirichlet_mask()[: 3 * nn], prec)
        assert np.array_equal(ia, ib)
        assert np.array_equal(port.bj_apply(ia, prec, u), reference.bj_apply(ib, prec, u))


def test_transfers_bit_exact(port, reference):
    m = reference.box_mesh((1.0, 2.0, 1.0), (2, 3, 2), (), 1)
    x = reference.rng_sym(3, 3 * m.vertex_count * 4).reshape(-1, 4)
    assert np.array_equal(port.geo_prolong(m, x, False), reference.geo_prolong(m, x, False))
    y = reference.rng_sym(4, 3 * m.n_nodes * 4).reshape(-1, 4)
    assert np.array_equal(port.geo_prolong(m, y, True), reference.geo_prolong(m, y, True))


@pytest.mark.parametrize("order", [1, 2])
def test_inner_pcg_bit_exact(port, reference, order):
    m = reference.box_mesh((400.0, 400.0, 200.0), (3, 3, 3), (100.0,), 1)
    lam, mu = lame(TWO_LAYER)
    nn = m.vertex_count if order == 1 else m.n_nodes
    mask = m.dirichlet_mask()[: 3 * nn]
    r = reference.rng_sym(7, 3 * nn * 3).reshape(-1, 3).astype(np.float32)
    r[mask == 1] = 0
    for tol, it in ((0.1, 30), (1e-4, 500)):
        a = port.inner_pcg_ebe(m, order, lam, mu, mask, r, np.zeros_like(r), tol, it)
        b = reference.inner_pcg_ebe(m, order, lam, mu, mask, r, np.zeros_like(r), tol, it)
        assert a[1:] == b[1:]
        assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("spec,batch", [(((400.0, 400.0, 200.0), (3, 3, 2), (100.0,), 1), 2),
                                        (((100.0, 100.0, 100.0), (2, 2, 2), (), 1), 3)])
def test_solve_bit_exact(port, reference, spec, batch):
    m = reference.box_mesh(*spec)
    lam, mu = lame(TWO_LAYER if spec[2] else STIFF)
    cfg = SolverConfig.default(batch_size=batch)
    la, lb = port.levels(m, lam, mu, cfg), reference.levels(m, lam, mu, cfg)
    ea, eb = la.export(), lb.export()
    for k in ea:
        assert np.array_equal(ea[k], eb[k]), k
    mask = m.dirichlet_mask()
    us = reference.rng_sym(9, 3 * m.n_nodes * batch).reshape(-1, batch)
    us[mask == 1] = 0
    f = lb.outer_apply(us)
    assert np.array_equal(la.outer_apply(us), f)
    ua, ra = la.solve(f, history=100)
    ub, rb = lb.solve(f, history=100)
    assert ra["outer_iterations"] == rb["outer_iterations"]
    assert ra["inner_iterations"] == rb["inner_iterations"]
    assert np.array_equal(ua, ub)
    assert np.array_equal(ra["history"], rb["history"])
    assert np.array_equal(ra["final_rel_residual"], rb["final_rel_residual"])
    pa, qa = la.solve_pcge(f)
    pb, qb = lb.solve_pcge(f)
    assert qa["outer_iterations"] == qb["outer_iterations"]
    assert np.array_equal(pa, pb)


def test_convergence_error_carries_report(port, reference):
    m = reference.box_mesh((400.0, 400.0, 200.0), (3, 3, 2), (100.0,), 1)
    lam, mu = lame(TWO_LAYER)
    cfg = SolverConfig.default(batch_size=1, outer_max_iter=1)
    for o in (port, reference):
        lv = o.levels(m, lam, mu, cfg)
        us = reference.rng_sym(5, 3 * m.n_nodes).reshape(-1, 1)
        us[m.dirichlet_mask() == 1] = 0
        with pytest.raises(Exception) as ei:
            lv.solve(lv.outer_apply(us))
        assert ei.value.code == 4
        assert ei.value.report["outer_iterations"] == 1
        assert not ei.value.report["converged"]


# ---------------------------------------------------------- golden fixtures
def _golden_mesh(g):
    return MeshArrays(g["coords"], g["tets10"], g["material_id"], int(g["vertex_count"]), g["bc_node"],
                      g["bc_axis"])


def test_port_matches_golden_ebe(port):
    g = np.load(os.path.join(GOLD, "ebe_2x2x2.npz"))
    m = _golden_mesh(g)
    a = port.box_mesh((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1)
    assert np.array_equal(a.coords, m.coords) and np.array_equal(a.tets10, m.tets10)
    mask = m.dirichlet_mask()
    for prec in (32, 64):
        for order in (1, 2):
            nn = m.vertex_count if order == 1 else m.n_nodes
            f = port.ebe_apply(m, order, g["lam"], g["mu"], mask[: 3 * nn], prec, g[f"u_{prec}_{order}"])
            assert np.array_equal(f, g[f"f_{prec}_{order}"])
            bj = port.ebe_block_jacobi(m, order, g["lam"], g["mu"], mask[: 3 * nn], prec)
            assert np.array_equal(bj, g[f"bj_{prec}_{order}"])


def test_port_matches_golden_solve(port):
    g = np.load(os.path.join(GOLD, "solve_4x4x4.npz"))
    m = port.box_mesh((400.0, 400.0, 200.0), (4, 4, 4), (100.0,), 1)
    lam, mu = lame(TWO_LAYER)
    lv = port.levels(m, lam, mu, SolverConfig.default(batch_size=2))
    ex = lv.export()
    assert lv.n2 == int(g["n2"])
    assert np.array_equal(ex["agg"], g["agg"])
    assert np.array_equal(ex["blocks2"], g["blocks2"])
    u, rep = lv.solve(g["f"], history=200)
    assert rep["outer_iterations"] == int(g["outer"])
    assert rep["inner_iterations"] == list(g["inner"])
    assert np.array_equal(u, g["u"])
    assert np.array_equal(rep["history"], g["history"])
    up, rp = lv.solve_pcge(g["f"])
    assert rp["outer_iterations"] == int(g["pcge_outer"])
    assert np.array_equal(up, g["u_pcge"])
