"""Parity on an UNSTRUCTURED mesh: the box generator's mesh with jittered interior
vertices (edge nodes kept at the new midpoints), random per-element materials,
shuffled element order and shuffled node numbering (vertices kept a prefix, as
mesh.hpp:26-42 requires). Every element then has its own shape and the node
numbering has no locality, so the pair matching / relabelling, the element order,
the host-buffer streaming schedule and the partitioned plans run off the
structured-mesh happy path. The checker is the reference compiled in place (else
the pinned port); tolerances are the north-star's (matvec 1e-5 / 1e-12, u 1e-6,
iteration counts +-2 %)."""
import threading

import numpy as np
import pytest
from conftest import TWO_LAYER, lame

import paper_1710_08679_b200 as ts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EDGES = ((0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3))


def scrambled_mesh(checker, ext, div, seed, jitter=0.1):
    """MeshArrays of a jittered, renumbered, reordered box mesh (and the product Mesh of it)."""
    from oracle import MeshArrays
    a = checker.box_mesh(ext, div, (0.5 * ext[2],), 1)
    rng = np.random.default_rng(seed)
    coords = a.coords.copy()
    V, N = a.vertex_count, a.n_nodes
    h = np.array(ext) / np.array(div)
    vx = coords[:V]
    interior = np.all((vx > 1e-9 * np.array(ext)) & (vx < np.array(ext) * (1 - 1e-9)), axis=1)
    vx[interior] += rng.uniform(-jitter, jitter, (int(interior.sum()), 3)) * h
    t = a.tets10.astype(np.int64)
    for k, (p, q) in enumerate(EDGES):  # edge nodes back at the midpoints of their (moved) ends
        coords[t[:, 4 + k]] = 0.5 * (coords[t[:, p]] + coords[t[:, q]])
    # node renumbering: vertices among themselves, edge nodes among themselves
    new = np.empty(N, np.int64)
    new[:V] = rng.permutation(V)
    new[V:] = V + rng.permutation(N - V)
    c2 = np.empty_like(coords)
    c2[new] = coords
    order = rng.permutation(len(t))
    tets = new[t][order].astype(np.int32)
    mat = rng.integers(0, 2, len(t)).astype(np.int32)
    m = MeshArrays(c2, tets, mat, V, new[a.bc_node].astype(np.int32), a.bc_axis.copy())
    # every element keeps a positive volume
    x = m.coords[m.tets10[:, :4].astype(np.int64)]
    vol = np.einsum("ij,ij->i", x[:, 1] - x[:, 0], np.cross(x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]))
    assert (vol > 0).all()
    pm = ts.Mesh.from_arrays(m.coords, m.tets10, m.material_id, V, m.bc_node, m.bc_axis)
    return m, pm


def mats():
    return [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def meshes(checker):
    return scrambled_mesh(checker, (3000.0, 2000.0, 1500.0), (6, 5, 4), 5)


@pytest.mark.parametrize("kernel", ["auto", "pipe", "fast", "color", "fan"])
@pytest.mark.parametrize("order", [2, 1])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("batch", [1, 4, 16, 3])
def test_ebe_unstructured(checker, meshes, monkeypatch, kernel, order, prec, batch):
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    m, pm = meshes
    nn = m.vertex_count if order == 1 else m.n_nodes
    mask = m.dirichlet_mask()[: 3 * nn]
    lam, mu = lame(TWO_LAYER)
    op = ts.EbeOperator(pm, order, mats(), mask, prec=prec)
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(91 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(dt)
    want = checker.ebe_apply(m, order, lam, mu, mask, prec, u)
    got = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got, want) <= (1e-5 if prec == 32 else 1e-12)
    assert np.array_equal(got[mask == 1], u[mask == 1])


@pytest.mark.parametrize("prec", [32, 64])
def test_host_streaming_unstructured(checker, prec):
    """A scrambled numbering: the streaming schedule's node blocks get no locality; still exact."""
    m, pm = scrambled_mesh(checker, (4000.0, 4000.0, 2000.0), (36, 36, 18), 9)
    op = ts.EbeOperator(pm, 2, mats(), m.dirichlet_mask(), prec=prec)
    dt = torch.float32 if prec == 32 else torch.float64
    u = torch.rand(3 * m.n_nodes, 16, device="cuda", dtype=dt) * 2 - 1
    fd = op.apply(u)
    uh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    uh.copy_(u.cpu())
    fh = torch.full(u.shape, float("nan"), dtype=dt, pin_memory=True)
    op.apply(uh.numpy(), fh.numpy())
    assert torch.isfinite(fh).all()
    assert rel(fh.numpy(), fd.cpu().numpy()) <= (1e-6 if prec == 32 else 1e-14)


def test_solve_unstructured(checker, meshes):
    from oracle import SolverConfig as OCfg
    m, pm = meshes
    B = 4
    lam, mu = lame(TWO_LAYER)
    cfg = ts.SolverConfig(batch_size=B)
    model = ts.build_crust_model(pm, mats(), cfg)
    rng = np.random.default_rng(3)
    us = rng.standard_normal((3 * m.n_nodes, B)) * (1 - m.dirichlet_mask()[:, None])
    f = model.levels.outer.apply(torch.from_numpy(us).cuda()).cpu().numpy()
    u, rep = ts.solve(model.levels, f, np.zeros_like(f), cfg)
    ref = checker.levels(m, lam, mu, OCfg.default(batch_size=B))
    ur, rr = ref.solve(f, np.zeros_like(f))
    assert rep.outer_iterations == rr["outer_iterations"]
    for a, b in zip(rep.inner_iterations, rr["inner_iterations"]):
        assert abs(a - b) <= max(2, 0.02 * b)
    assert rel(u, ur) <= 1e-6


def test_partitioned_product_unstructured(meshes):
    from paper_1710_08679_b200.dist import Comm, DistEbeOperator, ThreadWorld, partition_rcb
    m, pm = meshes
    P = 3
    part = partition_rcb(pm, P)
    single = ts.EbeOperator(pm, 2, mats(), m.dirichlet_mask(), prec=64)
    u = torch.rand(3 * m.n_nodes, 4, device="cuda", dtype=torch.float64)
    want = single.apply(u).cpu().numpy()
    world = ThreadWorld(P)
    comms = [Comm.thread(world, r, 0) for r in range(P)]
    out, err = [None] * P, [None] * P

    def body(r):
        try:
            torch.cuda.set_device(0)
            op = DistEbeOperator(pm, 2, mats(), part, comms[r], prec=64)
            nodes = op.local_nodes()
            dofs = (3 * nodes[:, None] + np.arange(3)).ravel()
            ul = u[torch.from_numpy(dofs).cuda()].contiguous()
            fl = torch.empty_like(ul)
            op.apply(ul, fl)
            torch.cuda.synchronize()
            out[r] = (dofs, fl.cpu().numpy())
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for dofs, fl in out:
        assert rel(fl, want[dofs]) <= 1e-12


@pytest.mark.parametrize("kernel", ["fan", "pair"])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("batch", [1, 8, 16])
def test_ebe_holey_mesh(checker, meshes, monkeypatch, kernel, prec, batch):
    """A third of the elements removed at random: edge rings break into open fans of every
    length (and closed fans of other valences), faces lose their partners, some nodes touch
    no element. The fan cover / pair matching must still produce exactly K u."""
    from oracle import MeshArrays
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    m, _ = meshes
    keep = np.random.default_rng(3).random(len(m.tets10)) > 0.33
    h = MeshArrays(m.coords, np.ascontiguousarray(m.tets10[keep]), np.ascontiguousarray(m.material_id[keep]),
                   m.vertex_count, m.bc_node, m.bc_axis)
    pm = ts.Mesh.from_arrays(h.coords, h.tets10, h.material_id, h.vertex_count, h.bc_node, h.bc_axis)
    mask = h.dirichlet_mask()
    lam, mu = lame(TWO_LAYER)
    op = ts.EbeOperator(pm, 2, mats(), mask, prec=prec)
    st = op.unit_stats()
    assert st["kind"] == ("fans" if kernel == "fan" else "pairs")
    if kernel == "fan":
        assert 0.0 < st["closed_fraction"] < 1.0 and 4.0 < st["rows_per_element"] < 10.0
    dt = np.float32 if prec == 32 else np.float64
    u = checker.rng_sym(17 + batch, 3 * h.n_nodes * batch).reshape(3 * h.n_nodes, batch).astype(dt)
    want = checker.ebe_apply(h, 2, lam, mu, mask, prec, u)
    got = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got, want) <= (1e-5 if prec == 32 else 1e-12)
    assert np.array_equal(got[mask == 1], u[mask == 1])
