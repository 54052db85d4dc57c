"""GPU parity of the EBE operator (EbeOperator<T>::apply, ebe_operator.hpp:90-188).

The CUDA product is called through the C ABI (ts_ebe_create / ts_ebe_apply)
and compared with the checker (the reference compiled in place when present,
else the bit-pinned C port) on the same seeded inputs. Tolerances are the
north-star's: a single matvec within 1e-12 (fp64) / 1e-5 (fp32) relative L2.
Re-states test_ebe.cpp:40-324 (zero in/out, nullspace, masked identity rows,
batch vs single, symmetry, shape mismatch) on the device path.
"""
import numpy as np
import pytest
from conftest import STIFF, TWO_LAYER, lame

import paper_1710_08679_b200 as ts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {32: 1e-5, 64: 1e-12}


def mats(table):
    return [ts.material_from_wavespeeds(*t) for t in table]


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


CASES = [
    (((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1), TWO_LAYER),
    (((400.0, 400.0, 200.0), (4, 3, 3), (100.0,), 1), TWO_LAYER),
    (((1.0, 1.0, 1.0), (2, 2, 1), (), 2), STIFF),
    (((3.0, 1.0, 2.0), (3, 1, 2), (), 0), STIFF),
]


KERNELS = ["auto", "pipe", "fast", "color", "pair", "fan"]  # TSGPU_EBE_KERNEL: default dispatch, generic and
# batch-specialised element-parallel RED sweeps, deterministic colored sweep, face-pair sweep, edge-fan sweep


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("batch", [1, 3, 4, 16, 20])
def test_ebe_matches_reference(checker, monkeypatch, kernel, case, prec, order, batch):
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    spec, table = case
    mesh = ts.generate_box_mesh(*spec)
    om = checker.box_mesh(*spec)
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    lam, mu = lame(table)
    op = ts.EbeOperator(mesh, order, mats(table), mask, prec=prec)
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(11 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(dt)
    want = checker.ebe_apply(om, order, lam, mu, mask, prec, u)
    got = op.apply(dev(u)).cpu().numpy()
    assert rel_l2(got, want) <= TOL[prec]
    # constrained dofs are identity rows, exactly (ebe_operator.hpp:96-110)
    assert np.array_equal(got[mask == 1], u[mask == 1])
    # host-buffer entry point gives the same numbers
    got_h = op.apply(u)
    assert rel_l2(got_h, want) <= TOL[prec]


@pytest.mark.parametrize("prec", [32, 64])
def test_zero_in_zero_out(prec):
    m = ts.generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 1))
    op = ts.EbeOperator(m, 2, mats(STIFF), m.dirichlet_mask(), prec=prec)
    dt = torch.float32 if prec == 32 else torch.float64
    f = op.apply(torch.zeros(3 * m.node_count(), 4, dtype=dt, device="cuda"))
    assert torch.count_nonzero(f).item() == 0


def test_rigid_translation_nullspace(checker):
    """test_ebe.cpp:48-75: unconstrained operator annihilates translations."""
    m = ts.generate_box_mesh((2.0, 2.0, 2.0), (2, 2, 2), (), 0)
    om = checker.box_mesh((2.0, 2.0, 2.0), (2, 2, 2), (), 0)
    lam, mu = lame(TWO_LAYER)
    k = checker.element_matrix(2, om.coords[om.tets10[0, :4]].ravel(), lam[1], mu[1])
    kscale = np.abs(k).max()
    for prec, tol in ((64, 1e-11), (32, 1e-5)):
        op = ts.EbeOperator(m, 2, mats(TWO_LAYER[1:]), None, prec=prec)
        dt = torch.float32 if prec == 32 else torch.float64
        for axis in range(3):
            t = torch.zeros(m.node_count(), 3, 1, dtype=dt, device="cuda")
            t[:, axis] = 1.0
            f = op.apply(t.reshape(-1, 1))
            assert f.abs().max().item() <= tol * kscale


def test_batched_columns_match_single_column_products():
    """test_ebe.cpp:254-269 (bit-exact there; the atomic scatter is
    order-nondeterministic, so equality is to fp64 rounding here)."""
    m = ts.generate_box_mesh((2.0, 2.0, 1.0), (2, 2, 1), (1.0 / 2,), 1)
    op = ts.EbeOperator(m, 2, mats(TWO_LAYER), m.dirichlet_mask(), prec=64)
    rng = np.random.default_rng(17)
    u = rng.uniform(-1, 1, (3 * m.node_count(), 16))
    f = op.apply(dev(u)).cpu().numpy()
    for b in range(16):
        fb = op.apply(dev(u[:, b:b + 1].copy())).cpu().numpy()[:, 0]
        assert rel_l2(fb, f[:, b]) < 1e-14


def test_operator_symmetry_fp32():
    """test_ebe.cpp:271-294."""
    m = ts.generate_box_mesh((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1)
    op = ts.EbeOperator(m, 2, mats(TWO_LAYER), m.dirichlet_mask(), prec=32)
    rng = np.random.default_rng(19)
    for _ in range(4):
        u = rng.uniform(-1, 1, (3 * m.node_count(), 1)).astype(np.float32)
        v = rng.uniform(-1, 1, (3 * m.node_count(), 1)).astype(np.float32)
        au, av = op.apply(u), op.apply(v)
        vau = float(np.dot(v[:, 0].astype(np.float64), au[:, 0]))
        uav = float(np.dot(u[:, 0].astype(np.float64), av[:, 0]))
        scale = np.linalg.norm(u) * np.linalg.norm(v) * np.abs(au).max()
        assert abs(vau - uav) <= 1e-6 * scale


def test_dimension_mismatch_rejected():
    """test_ebe.cpp:319-324."""
    m = ts.generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 1))
    op = ts.EbeOperator(m, 2, mats(STIFF), m.dirichlet_mask(), prec=64)
    with pytest.raises(ts.ValidationError):
        op.apply(torch.zeros(3 * m.node_count() + 3, 1, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("order", [1, 2])
def test_block_jacobi_matches_reference(checker, prec, order):
    spec = ((400.0, 400.0, 200.0), (3, 3, 2), (100.0,), 1)
    m = ts.generate_box_mesh(*spec)
    om = checker.box_mesh(*spec)
    nn = m.vertex_count if order == 1 else m.node_count()
    mask = m.dirichlet_mask()[: 3 * nn]
    lam, mu = lame(TWO_LAYER)
    op = ts.EbeOperator(m, order, mats(TWO_LAYER), mask, prec=prec)
    got = op.block_jacobi()
    want = checker.ebe_block_jacobi(om, order, lam, mu, mask, prec)
    assert rel_l2(got, want) <= (1e-6 if prec == 32 else 1e-12)


@pytest.mark.parametrize("batch", [8, 16])
def test_full_size_properties(batch):
    """Config-2 mesh (82x123x41 cells, ~10M DOF): size-independent checks —
    fp32 tier agrees with the fp64 tier (itself checked against the reference
    above) to 1e-5, linearity, and symmetry."""
    m = ts.generate_box_mesh((82e3, 123e3, 41e3), (82, 123, 41), (20e3,), 1)
    mk = m.dirichlet_mask()
    op32 = ts.EbeOperator(m, 2, mats(TWO_LAYER), mk, prec=32)
    op64 = ts.EbeOperator(m, 2, mats(TWO_LAYER), mk, prec=64)
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(3 * m.node_count(), batch, device="cuda", generator=g, dtype=torch.float32) * 2 - 1
    v = torch.rand(3 * m.node_count(), batch, device="cuda", generator=g, dtype=torch.float32) * 2 - 1
    f32 = op32.apply(u)
    f64 = op64.apply(u.double())
    assert ((f32.double() - f64).norm() / f64.norm()).item() <= 1e-5
    lin = op64.apply(u.double() + v.double()) - f64 - op64.apply(v.double())
    assert (lin.norm() / f64.norm()).item() <= 1e-13
    vau = (v.double() * f64).sum(0)
    uav = (u.double() * op64.apply(v.double())).sum(0)
    assert ((vau - uav).abs().max() / vau.abs().max()).item() <= 1e-10


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("prec,batch", [(32, 16), (32, 4), (64, 8)])
@pytest.mark.parametrize("order", [1, 2])
def test_ebe_many_chunks_per_block(checker, monkeypatch, kernel, prec, batch, order):
    """A mesh with many more element chunks than resident blocks, so every
    persistent block walks several chunks (pipelined record prefetch)."""
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    spec = ((6000.0, 5000.0, 4000.0), (24, 20, 16), (3000.0,), 1)
    mesh = ts.generate_box_mesh(*spec)
    om = checker.box_mesh(*spec)
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    lam, mu = lame(TWO_LAYER)
    op = ts.EbeOperator(mesh, order, mats(TWO_LAYER), mask, prec=prec)
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(5 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(dt)
    want = checker.ebe_apply(om, order, lam, mu, mask, prec, u)
    got = op.apply(dev(u)).cpu().numpy()
    assert rel_l2(got, want) <= TOL[prec]
    assert np.array_equal(got[mask == 1], u[mask == 1])


@pytest.mark.parametrize("kernel", ["auto", "fan"])
@pytest.mark.parametrize("order", [2, 1])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("batch", [1, 4, 16, 3])
def test_host_apply_streams_and_matches_device(monkeypatch, kernel, order, prec, batch):
    """ts_ebe_apply_host with pinned buffers overlaps H2D / sweep / D2H chunk by
    chunk (ebe_stream.cu): same f as the device apply, every row copied back;
    batch 3 (no pair / fan kernel) and pageable buffers take copy-apply-copy."""
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    cells = (40, 40, 20) if order == 2 else (60, 60, 30)
    mesh = ts.generate_box_mesh((4000.0, 4000.0, 2000.0), cells, (1200.0,))
    nn = mesh.node_count() if order == 2 else mesh.vertex_count
    op = ts.EbeOperator(mesh, order, mats(TWO_LAYER), mesh.dirichlet_mask()[: 3 * nn], prec=prec)
    dt = torch.float32 if prec == 32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(3 * nn, batch, device="cuda", dtype=dt, generator=g) * 2 - 1
    f_dev = op.apply(u)
    uh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    uh.copy_(u.cpu())
    fh = torch.full(u.shape, float("nan"), dtype=dt, pin_memory=True)
    op.apply(uh.numpy(), fh.numpy())
    assert op.host_stream_chunks() >= 2  # the schedule exists (batch 3 then falls back inside the call)
    got = fh.cuda()
    assert torch.isfinite(got).all()
    rel = float((got.double() - f_dev.double()).norm() / f_dev.double().norm())
    assert rel <= (1e-6 if prec == 32 else 1e-14)
    mask = torch.from_numpy(mesh.dirichlet_mask()[: 3 * nn].astype(bool)).cuda()
    assert torch.equal(got[mask], u[mask])  # identity rows exact
    # pageable buffers: copy-apply-copy, same answer
    fp = op.apply(u.cpu().numpy())
    assert float((torch.from_numpy(fp).cuda().double() - f_dev.double()).norm() / f_dev.double().norm()) <= (
        1e-6 if prec == 32 else 1e-14)


_SPLIT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/oracle'); sys.path.insert(0, sys.argv[1] + '/tests')
import paper_1710_08679_b200 as ts
from conftest import TWO_LAYER, lame
from oracle import Oracle, have_reference
chk = Oracle('reference' if have_reference() else 'port')
spec = ((4000.0, 3000.0, 2000.0), (40, 30, 20), (1000.0,), 1)
mesh, om = ts.generate_box_mesh(*spec), chk.box_mesh(*spec)
lam, mu = lame(TWO_LAYER)
worst = 0.0
for prec, order, batch in ((32, 2, 16), (32, 1, 4), (64, 2, 8), (32, 2, 1)):
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    op = ts.EbeOperator(mesh, order, [ts.material_from_wavespeeds(*t) for t in TWO_LAYER], mask, prec=prec)
    dt = np.float32 if prec == 32 else np.float64
    u = chk.rng_sym(5 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(dt)
    want = chk.ebe_apply(om, order, lam, mu, mask, prec, u)
    got = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    r = float(np.linalg.norm(got.astype(np.float64) - want) / np.linalg.norm(want))
    worst = max(worst, r / (1e-5 if prec == 32 else 1e-12))
print(worst)
"""


@pytest.mark.parametrize("dyn", ["1", "0"])
@pytest.mark.parametrize("strides", ["1", "3", None])
def test_pair_sweep_split_into_many_launches(strides, dyn):
    """TSGPU_EBE_PAIR_STRIDES / TSGPU_EBE_DYN (read once per process, so in a child
    process): a sweep split into launches of 1 or 3 grid strides each (up to ~30
    launches here), with the dynamic unit schedule (a counter per launch) or the static
    strides, gives the reference's product, as the single-launch sweep does."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSGPU_EBE_DYN=dyn, TSGPU_EBE_KERNEL="pair")
    env.pop("TSGPU_EBE_PAIR_STRIDES", None)
    if strides is not None:
        env["TSGPU_EBE_PAIR_STRIDES"] = strides
    out = subprocess.run([sys.executable, "-c", _SPLIT_SCRIPT, root], capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1.0


@pytest.mark.parametrize("prec", [32, 64])
def test_concurrent_applies_on_streams(prec):
    """One operator applied concurrently on four CUDA streams (the pair sweep's dynamic
    schedule gives each launch its own unit counter, ebe_pair.cu): every product equals the
    one computed alone."""
    mesh = ts.generate_box_mesh((3000.0, 3000.0, 2000.0), (24, 24, 16), (900.0,))
    op = ts.EbeOperator(mesh, 2, mats(TWO_LAYER), mesh.dirichlet_mask(), prec=prec)
    dt = torch.float32 if prec == 32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(11)
    us = [torch.rand(3 * op.n_nodes(), 16, device="cuda", dtype=dt, generator=g) * 2 - 1 for _ in range(4)]
    alone = [op.apply(u) for u in us]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in us]
    outs = [torch.empty_like(u) for u in us]
    for _ in range(3):
        for st, u, f in zip(streams, us, outs):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                op.apply(u, f)
        torch.cuda.synchronize()
        for f, a in zip(outs, alone):
            assert rel_l2(f.double().cpu().numpy(), a.double().cpu().numpy()) <= TOL[prec]
