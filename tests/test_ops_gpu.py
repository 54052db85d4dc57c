"""Op-level device parity of the solve path's building blocks against the
reference (the checker: oracle/_ref when built, else the pinned C port).

* the standalone operators of the drop-in boundary (ts_bcsr_*, ts_bj_*,
  ts_prolong_*, ts_inner_pcg, ts_ebe_element_matrix, ts_ebe_assemble_bcsr):
  BlockCsrMatrix::apply (block_csr.hpp:33-69) and the transfers
  (prolongation.hpp:25-61) bit-exact, element matrices / assembly at fp64
  rounding, inner_pcg (pcg.hpp:52-124) iteration counts and iterates;
* the kernels the multigrid solve itself runs (ts_levels_apply which = 3: the
  level-2 SpMV; ts_levels_transfer: P1, P1^T, P2, P2^T with their masks);
* the reference's error paths: an indefinite operator raises SolverError
  (test_solver.cpp:123-135), a non-finite residual raises SolverError
  (pcg.hpp:70,118-120; adaptive_cg.hpp:171);
* the deterministic (colored) sweep: batched columns equal single-column
  products bit for bit and repeated applies are bitwise identical
  (test_ebe.cpp:254-269, :296-317).
"""
import numpy as np
import pytest
from conftest import STIFF, TWO_LAYER, lame

import paper_1710_08679_b200 as ts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPEC = ((16000.0, 20000.0, 10000.0), (5, 6, 4), (7000.0,), 1)


def mats(table):
    return [ts.material_from_wavespeeds(*t) for t in table]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def box(checker):
    mesh = ts.generate_box_mesh(*SPEC)
    om = checker.box_mesh(*SPEC)
    return mesh, om


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("prec", [32, 64])
def test_assemble_bcsr_and_bcsr_apply(checker, box, order, prec):
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    op = ts.EbeOperator(mesh, order, mats(TWO_LAYER), mask, prec=prec)
    a = ts.assemble_bcsr(op)
    rp, ci, bl = checker.assemble_bcsr(om, order, lam, mu, mask, prec)
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)  # same pattern
    assert rel(a.blocks, bl) <= (1e-6 if prec == 32 else 1e-13)
    # BlockCsrMatrix::apply: fp64 row sums in stored order, rounded to T -> bit-exact on the same blocks
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(7, 3 * nn * 5).reshape(3 * nn, 5).astype(dt)
    want = checker.bcsr_apply(rp, ci, a.blocks, prec, u)
    assert np.array_equal(a.apply(u), want)
    assert np.array_equal(a.apply(torch.from_numpy(u).cuda()).cpu().numpy(), want)
    # EBE equals its assembled matrix (test_ebe.cpp:77-111)
    f = op.apply(u)
    assert rel(f, want) <= (1e-5 if prec == 32 else 1e-13)


@pytest.mark.parametrize("order", [1, 2])
def test_element_matrix_matches_reference(checker, box, order):
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    op = ts.EbeOperator(mesh, order, mats(TWO_LAYER), None, prec=64)
    for e in (0, 7, mesh.element_count() - 1):
        v12 = om.coords[om.tets10[e, :4]].reshape(-1)
        mid = om.material_id[e]
        want = checker.element_matrix(order, v12, lam[mid], mu[mid])
        got = op.element_matrix(e)
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
        assert np.allclose(got, got.T, rtol=0, atol=1e-14 * np.abs(got).max())


@pytest.mark.parametrize("prec", [32, 64])
def test_block_jacobi_apply_and_bcsr_extraction(checker, box, prec):
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    mask = mesh.dirichlet_mask()
    op = ts.EbeOperator(mesh, 2, mats(TWO_LAYER), mask, prec=prec)
    inv = op.block_jacobi()
    m = ts.BlockJacobi(inv)
    dt = np.float32 if prec == 32 else np.float64
    r = checker.rng_sym(9, 3 * mesh.node_count() * 3).reshape(-1, 3).astype(dt)
    want = checker.bj_apply(inv, prec, r)
    got = m.apply(r)
    assert rel(got, want) <= (1e-7 if prec == 32 else 1e-15)
    # extract_block_jacobi(assemble_bcsr(op)) = extract_block_jacobi(op) (block_jacobi.hpp:72-85 vs ebe_operator.hpp:288)
    bj2 = ts.assemble_bcsr(op).block_jacobi()
    assert rel(bj2.inv_blocks, inv) <= (1e-5 if prec == 32 else 1e-12)


def test_geometric_prolongation_bit_exact(checker, box):
    mesh, om = box
    p = ts.build_geometric_prolongation(mesh)
    assert p.n_fine_nodes == mesh.node_count() and p.n_coarse_nodes == mesh.vertex_count
    xc = checker.rng_sym(3, 3 * mesh.vertex_count * 4).reshape(-1, 4).astype(np.float32)
    xf = checker.rng_sym(4, 3 * mesh.node_count() * 4).reshape(-1, 4).astype(np.float32)
    assert np.array_equal(p.apply(xc), checker.geo_prolong(om, xc, False))
    assert np.array_equal(p.restrict_to_coarse(xf), checker.geo_prolong(om, xf, True))
    assert np.array_equal(p.apply(torch.from_numpy(xc).cuda()).cpu().numpy(), checker.geo_prolong(om, xc, False))


@pytest.fixture(scope="module")
def levels(checker, box):
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    from oracle import SolverConfig as OCfg
    lv = ts.build_crust_model(mesh, mats(TWO_LAYER), ts.SolverConfig(batch_size=4)).levels
    olv = checker.levels(om, lam, mu, OCfg.default(batch_size=4))
    return lv, olv


@pytest.mark.parametrize("batch", [1, 4, 16])
def test_solver_level2_spmv(checker, levels, batch):
    """The level-2 SpMV the preconditioner runs (k_bcsr_rows, fp64 row sums) vs BlockCsrMatrix::apply."""
    lv, _ = levels
    ex = lv.export()
    u = checker.rng_sym(21, 3 * lv.n2 * batch).reshape(-1, batch).astype(np.float32)
    want = checker.bcsr_apply(ex["row_ptr2"], ex["col_idx2"], ex["blocks2"], 32, u)
    got = lv.apply(3, torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got, want) <= 1e-7
    assert np.abs(got - want).max() <= 4 * np.finfo(np.float32).eps * np.abs(want).max()


@pytest.mark.parametrize("batch", [1, 4, 16])
def test_solver_transfers_bit_exact(checker, box, levels, batch):
    """P1 / P1^T (geometric) and P2 / P2^T (aggregation) as the solve runs them, each with the
    zero_masked of its output level (adaptive_cg.hpp:84-107), against the reference's transfers."""
    mesh, om = box
    lv, _ = levels
    ex = lv.export()
    agg = ex["agg"]
    mask0 = mesh.dirichlet_mask()
    mask1 = mask0[: 3 * lv.n1]
    mask2 = ex["mask2"]
    g = lambda n, seed: checker.rng_sym(seed, 3 * n * batch).reshape(-1, batch).astype(np.float32)  # noqa: E731
    dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    x1, x0, x2 = g(lv.n1, 1), g(lv.n0, 2), g(lv.n2, 3)
    want = checker.geo_prolong(om, x1, False)
    want[mask0 == 1] = 0
    assert np.array_equal(lv.transfer(0, dev(x1)).cpu().numpy(), want)
    want = checker.geo_prolong(om, x0, True)
    want[mask1 == 1] = 0
    assert np.array_equal(lv.transfer(1, dev(x0)).cpu().numpy(), want)
    p2 = ts.Prolongation(lv.n1, lv.n2, np.arange(lv.n1 + 1), agg, np.ones(lv.n1))
    want = p2.apply(x2)
    want[mask1 == 1] = 0
    assert np.array_equal(lv.transfer(2, dev(x2)).cpu().numpy(), want)
    want = np.zeros((3 * lv.n2, batch), np.float32)  # serial scatter-add in ascending fine node order
    x1n = x1.reshape(lv.n1, 3, batch)
    w3 = want.reshape(lv.n2, 3, batch)
    for node in range(lv.n1):
        w3[agg[node]] += x1n[node]
    want[mask2 == 1] = 0
    assert np.array_equal(lv.transfer(3, dev(x1)).cpu().numpy(), want)
    assert np.array_equal(p2.restrict_to_coarse(x1)[mask2 == 0], want[mask2 == 0])


@pytest.mark.parametrize("batch", [1, 3])
def test_inner_pcg_ebe_matches_reference(checker, box, batch):
    """inner_pcg (pcg.hpp:52-124) on the fp32 tet10 operator with its block Jacobi: the
    reference's iteration count and iterate."""
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    mask = mesh.dirichlet_mask()
    op = ts.EbeOperator(mesh, 2, mats(TWO_LAYER), mask, prec=32)
    m = ts.BlockJacobi(op.block_jacobi())
    r = checker.rng_sym(62, 3 * mesh.node_count() * batch).reshape(-1, batch).astype(np.float32)
    r[mask == 1] = 0
    u0 = np.zeros_like(r)
    for tol, max_iter in ((0.1, 30), (1e-4, 400)):
        want, it_ref, conv_ref = checker.inner_pcg_ebe(om, 2, lam, mu, mask, r, u0, tol, max_iter)
        u = u0.copy()
        st = ts.inner_pcg(op, m, r, u, tol, max_iter)
        assert abs(st.iterations - it_ref) <= max(1, 0.02 * it_ref) and st.converged == conv_ref
        assert rel(u, want) <= 1e-4
        ud = torch.zeros(r.shape, dtype=torch.float32, device="cuda")
        st_d = ts.inner_pcg(op, m, torch.from_numpy(r).cuda(), ud, tol, max_iter)
        assert st_d.iterations == st.iterations


def test_inner_pcg_exact_preconditioner_one_step(checker):
    """test_solver.cpp:30-56: with M = A^-1 (block diagonal SPD), one step converges."""
    rng = np.random.default_rng(61)
    n = 6
    blocks = []
    for _ in range(n):
        b = rng.uniform(-1, 1, (3, 3))
        blocks.append((b @ b.T + 3 * np.eye(3)).astype(np.float32).reshape(9))
    a = ts.BlockCsrMatrix(n, np.arange(n + 1), np.arange(n), np.array(blocks, np.float32))
    m = a.block_jacobi()
    r = rng.uniform(-1, 1, (3 * n, 3)).astype(np.float32)
    u = np.zeros_like(r)
    st = ts.inner_pcg(a, m, r, u, 1e-5, 50)
    assert st.converged and st.iterations == 1


def test_inner_pcg_indefinite_operator_raises():
    """test_solver.cpp:123-135: (p, Ap) < 0 without stagnation is a breakdown -> SolverError."""
    a = ts.BlockCsrMatrix(2, [0, 1, 2], [0, 1],
                          np.array([[1, 0, 0, 0, 1, 0, 0, 0, 1], [-2, 0, 0, 0, -2, 0, 0, 0, -2]], np.float32))
    m = ts.BlockJacobi(np.array([[1, 0, 0, 0, 1, 0, 0, 0, 1]] * 2, np.float32))
    r = np.ones((6, 1), np.float32)
    u = np.zeros_like(r)
    with pytest.raises(ts.SolverError, match="breakdown"):
        ts.inner_pcg(a, m, r, u, 1e-10, 100)


def test_nonfinite_residual_raises():
    """pcg.hpp:70 (inner) and adaptive_cg.hpp:171 (outer): a NaN in the residual is a SolverError."""
    a = ts.BlockCsrMatrix(2, [0, 1, 2], [0, 1], np.array([[2, 0, 0, 0, 2, 0, 0, 0, 2]] * 2, np.float32))
    m = a.block_jacobi()
    r = np.ones((6, 2), np.float32)
    r[3, 1] = np.nan
    with pytest.raises(ts.SolverError, match="non-finite"):
        ts.inner_pcg(a, m, r, np.zeros_like(r), 1e-6, 10)
    mesh = ts.generate_box_mesh((100.0, 100.0, 100.0), (2, 2, 2))
    model = ts.build_crust_model(mesh, mats(STIFF), ts.SolverConfig(batch_size=2))
    f = np.random.default_rng(3).uniform(-1, 1, (3 * mesh.node_count(), 2))
    f[model.mask == 1] = 0
    f[-1, 0] = np.nan
    with pytest.raises(ts.SolverError, match="non-finite"):
        ts.solve(model.levels, f, np.zeros_like(f), ts.SolverConfig(batch_size=2))


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("order", [1, 2])
def test_deterministic_sweep_bitwise(checker, box, prec, order):
    """Colored sweep: bitwise reproducible, batched columns == single-column products,
    and the reference's product within the north-star tolerance."""
    mesh, om = box
    lam, mu = lame(TWO_LAYER)
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    op = ts.EbeOperator(mesh, order, mats(TWO_LAYER), mask, prec=prec).set_deterministic(True)
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(17, 3 * nn * 16).reshape(-1, 16).astype(dt)
    ud = torch.from_numpy(u).cuda()
    f1, f2 = op.apply(ud), op.apply(ud)
    assert torch.equal(f1, f2)
    for b in (0, 5, 15):
        fb = op.apply(ud[:, b:b + 1].contiguous())
        assert torch.equal(fb[:, 0], f1[:, b])
    f4 = op.apply(ud[:, :4].contiguous())
    assert torch.equal(f4, f1[:, :4])
    want = checker.ebe_apply(om, order, lam, mu, mask, prec, u)
    assert rel(f1.cpu().numpy(), want) <= (1e-5 if prec == 32 else 1e-12)
    assert op.launches_per_apply(16) >= 8  # one launch per color (+ init)
